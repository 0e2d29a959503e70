"""Build every native artefact in-tree without importing the product package:
libdpg.so (nvcc, sm_100a), oracle/liboracle.so and datagen/libdpggen.so (gcc)."""
from __future__ import annotations

import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(path: str, name: str):
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def build_dpg(force: bool = False) -> str:
    b = _load(os.path.join(ROOT, "paper_cs_0308004_b200", "build.py"), "_dpg_build")
    return b.build(force=force)


def build_all(force: bool = False) -> list[str]:
    import datagen
    import oracle
    return [build_dpg(force), oracle.build(force), datagen.build(force)]


if __name__ == "__main__":
    import sys
    sys.path.insert(0, ROOT)
    for p in build_all(force="--force" in sys.argv):
        print(p)
