"""CPU oracle for DPG record retrieval (arXiv cs/0308004) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
path (``paper_cs_0308004_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, single thread); this
module only compiles it with gcc and marshals numpy arrays through ctypes.
Each wrapper cites the passage the C function follows:

* :func:`retrieve`    -- the problem's definition ``D[i] = R[S_rid[i]]``
* :func:`dpg_fig1`    -- the three phases of Fig. 1, INTERNAL materialised
* :func:`fk_join`     -- DPG-Move join rows ``fact[i] ++ dim[fk[i]]``
* :func:`retrieve_at` -- the definition evaluated at sampled output positions
* :func:`retrieve_generated` -- the definition for a counter-generated source too
  large for the host (config 5), at sampled rows
* :func:`sort_rids`   -- phases 1-2 of three-phase key-pointer sorting:
  the rids in stable key order
* :func:`sort`        -- the whole three-phase sort: sort_rids then retrieve
* :func:`fk_join_sort` -- DPG-Sort join rows ``fact[rid_R] ++ dim[rid_F]`` in rid_F order
  

Errors (reading A6 in DESIGN.md): a rid >= n_src raises :class:`RidRangeError`
carrying the smallest offending position.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


class RidRangeError(ValueError):
    def __init__(self, index: int):
        super().__init__(f"rid out of range at position {index}")
        self.index = index


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (no CUDA; plain -O2, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", _SRC, "-o", tmp,
                               "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P, U = ctypes.c_void_p, ctypes.c_uint64
        lib.oracle_retrieve.argtypes = [P, U, U, P, U, P, P]
        lib.oracle_retrieve_u64.argtypes = [P, U, U, P, U, P, P]
        lib.oracle_retrieve_threads.argtypes = [P, U, U, P, U, P, P, ctypes.c_int]
        lib.oracle_retrieve_threads.restype = ctypes.c_int
        lib.oracle_dpg_fig1.argtypes = [P, U, U, P, U, U, P, P, P, P, P, P]
        lib.oracle_fk_join.argtypes = [P, U, U, P, P, U, U, P, P]
        lib.oracle_retrieve_at.argtypes = [P, U, U, P, P, U, P]
        lib.oracle_retrieve_at_u64.argtypes = [P, U, U, P, P, U, P]
        lib.oracle_retrieve_at_u64.restype = ctypes.c_int
        lib.oracle_sort_rids.argtypes = [P, U, U, U, U, P]
        lib.oracle_fk_join_sort.argtypes = [P, U, U, P, P, U, U, P, P]
        lib.oracle_batch_lookup.argtypes = [P, U, P, U, P]
        lib.oracle_batch_lookup.restype = ctypes.c_int
        lib.oracle_fk_join_sort.restype = ctypes.c_int
        lib.oracle_splitmix64.argtypes = [U, U]
        lib.oracle_splitmix64.restype = ctypes.c_uint64
        lib.oracle_skew_partition.argtypes = [P, U, U, U, U, U, P, P]
        lib.oracle_skew_partition.restype = ctypes.c_int
        lib.oracle_dpg_bounds.argtypes = [P, U, U, P, U, P, U, P, P, P, P]
        lib.oracle_dpg_bounds.restype = ctypes.c_int
        for f in (lib.oracle_retrieve, lib.oracle_retrieve_u64, lib.oracle_dpg_fig1,
                  lib.oracle_fk_join, lib.oracle_retrieve_at, lib.oracle_sort_rids):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _records(src: np.ndarray) -> np.ndarray:
    src = np.ascontiguousarray(src, dtype=np.uint8)
    if src.ndim == 1:
        src = src.reshape(-1, 1)
    return src


def _check(status: int, bad: ctypes.c_uint64):
    if status == -1:
        raise ValueError("invalid argument")
    if status == 1:
        raise RidRangeError(int(bad.value))


def retrieve(src: np.ndarray, rids: np.ndarray) -> np.ndarray:
    """D[i] = R[S_rid[i]].  src: uint8 [n_src, rec]; rids: uint32/uint64 [n_out]."""
    src = _records(src)
    n_src, rec = src.shape
    rids = np.ascontiguousarray(rids)
    if rids.dtype not in (np.uint32, np.uint64):
        if rids.size and (rids.min() < 0):
            raise RidRangeError(int(np.argmax(rids < 0)))
        rids = rids.astype(np.uint64)
    dst = np.zeros((rids.size, rec), dtype=np.uint8)
    bad = ctypes.c_uint64(0)
    fn = _load().oracle_retrieve if rids.dtype == np.uint32 else _load().oracle_retrieve_u64
    _check(fn(_ptr(src), rec, n_src, _ptr(rids), rids.size, _ptr(dst), ctypes.byref(bad)), bad)
    return dst


def retrieve_threads(src: np.ndarray, rids: np.ndarray, threads: int) -> np.ndarray:
    """The definition's loop split into `threads` contiguous index ranges, one
    host thread each (all-cores CPU baseline timing; uint32 rids)."""
    src = _records(src)
    n_src, rec = src.shape
    rids = np.ascontiguousarray(rids, dtype=np.uint32)
    dst = np.zeros((rids.size, rec), dtype=np.uint8)
    bad = ctypes.c_uint64(0)
    _check(_load().oracle_retrieve_threads(_ptr(src), rec, n_src, _ptr(rids), rids.size, _ptr(dst),
                                           ctypes.byref(bad), int(threads)), bad)
    return dst


def retrieve_at(src: np.ndarray, rids: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Rows D[idx[j]] of the definition, for sampled parity at full sizes
    (uint32 or uint64 rids; no cast)."""
    src = _records(src)
    n_src, rec = src.shape
    rids = np.ascontiguousarray(rids)
    if rids.dtype not in (np.uint32, np.uint64):
        rids = rids.astype(np.uint64)
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.zeros((idx.size, rec), dtype=np.uint8)
    fn = _load().oracle_retrieve_at if rids.dtype == np.uint32 else _load().oracle_retrieve_at_u64
    if fn(_ptr(src), rec, n_src, _ptr(rids), _ptr(idx), idx.size, _ptr(out)):
        raise RidRangeError(-1)
    return out


def retrieve_generated(rec: int, n_src: int, sid: int, rids: np.ndarray,
                       seed: int = 0) -> np.ndarray:
    """D[i] = R[rids[i]] for a source R too large to hold on the
    host (config 5: 2^30 x 100 B) whose record r is bytes [r*rec, (r+1)*rec)
    of the counter-based stream sid (datagen, reading A12): each needed record
    is generated at its offset and handed to oracle_retrieve_u64 as a compact
    source.  For sampled rows only (a Python loop over the rids)."""
    import datagen
    rids = np.ascontiguousarray(rids).astype(np.uint64)
    bad = np.nonzero(rids >= np.uint64(n_src))[0]
    if bad.size:
        raise RidRangeError(int(bad[0]))
    uniq, inv = np.unique(rids, return_inverse=True)
    compact = np.stack([datagen.random_bytes(rec, sid, seed=seed, offset=int(r) * rec)
                        for r in uniq]) if uniq.size else np.zeros((0, rec), np.uint8)
    return retrieve(compact, inv.astype(np.uint64))


def dpg_fig1(src: np.ndarray, rids: np.ndarray, L: int):
    """Fig. 1's three phases.  Returns a dict with ``dst`` and the
    intermediates ``run_start`` (NUM_RUNS+1), ``rid_runs`` (RID_RUN[0]++...),
    ``rid_pos`` (source position of each RID_RUN entry) and ``record_runs``
    (INTERNAL = RECORD_RUN[0]++...)."""
    src = _records(src)
    n_src, rec = src.shape
    rids = np.ascontiguousarray(rids, dtype=np.uint32)
    n_out = rids.size
    num_runs = (n_src + L - 1) // L
    dst = np.zeros((n_out, rec), dtype=np.uint8)
    run_start = np.zeros(num_runs + 1, dtype=np.uint64)
    rid_runs = np.zeros(n_out, dtype=np.uint32)
    rid_pos = np.zeros(n_out, dtype=np.uint64)
    record_runs = np.zeros((n_out, rec), dtype=np.uint8)
    bad = ctypes.c_uint64(0)
    st = _load().oracle_dpg_fig1(_ptr(src), rec, n_src, _ptr(rids), n_out, L, _ptr(dst),
                                 _ptr(run_start), _ptr(rid_runs), _ptr(rid_pos),
                                 _ptr(record_runs), ctypes.byref(bad))
    _check(st, bad)
    return {"dst": dst, "run_start": run_start, "rid_runs": rid_runs,
            "rid_pos": rid_pos, "record_runs": record_runs}


def fk_join(fact: np.ndarray, fk: np.ndarray, dim: np.ndarray) -> np.ndarray:
    """DPG-Move join rows ``fact[i] ++ dim[fk[i]]`` in fact order (reading A11)."""
    fact = _records(fact)
    dim = _records(dim)
    n_fact, fact_bytes = fact.shape
    n_dim, rec = dim.shape
    fk = np.ascontiguousarray(fk, dtype=np.uint32)
    assert fk.size == n_fact
    out = np.zeros((n_fact, fact_bytes + rec), dtype=np.uint8)
    bad = ctypes.c_uint64(0)
    _check(_load().oracle_fk_join(_ptr(fact), fact_bytes, n_fact, _ptr(fk), _ptr(dim), rec,
                                  n_dim, _ptr(out), ctypes.byref(bad)), bad)
    return out


def sort_rids(src: np.ndarray, key_off: int, key_bytes: int) -> np.ndarray:
    """Phases 1-2 of three-phase sorting: the rids of the records
    in stable order of their key (key_bytes unsigned bytes at key_off)."""
    src = _records(src)
    n, rec = src.shape
    out = np.zeros(n, dtype=np.uint32)
    if _load().oracle_sort_rids(_ptr(src), rec, n, key_off, key_bytes, _ptr(out)):
        raise ValueError("invalid argument")
    return out


def sort(src: np.ndarray, key_off: int, key_bytes: int) -> np.ndarray:
    """The three-phase key-pointer sort: sorted records."""
    return retrieve(src, sort_rids(src, key_off, key_bytes))


def fk_join_sort(fact: np.ndarray, fk: np.ndarray, dim: np.ndarray) -> np.ndarray:
    """DPG-Sort join rows ``fact[rid_R] ++ dim[rid_F]`` with the pairs in stable
    rid_F (= fk) order (reading A11)."""
    fact = _records(fact)
    dim = _records(dim)
    n_fact, fact_bytes = fact.shape
    n_dim, rec = dim.shape
    fk = np.ascontiguousarray(fk, dtype=np.uint32)
    assert fk.size == n_fact
    out = np.zeros((n_fact, fact_bytes + rec), dtype=np.uint8)
    bad = ctypes.c_uint64(0)
    _check(_load().oracle_fk_join_sort(_ptr(fact), fact_bytes, n_fact, _ptr(fk), _ptr(dim), rec,
                                       n_dim, _ptr(out), ctypes.byref(bad)), bad)
    return out



NOT_FOUND = 0xFFFFFFFF


def batch_lookup(keys: np.ndarray, queries: np.ndarray) -> np.ndarray:
    """Batch index lookup: out[i] = j with keys[j] == queries[i]
    (keys distinct), NOT_FOUND if none -- sorted pairs and binary search."""
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    q = np.ascontiguousarray(queries, dtype=np.uint32)
    out = np.empty(q.size, dtype=np.uint32)
    if _load().oracle_batch_lookup(_ptr(keys), keys.size, _ptr(q), q.size, _ptr(out)) != 0:
        raise ValueError("invalid argument")
    return out


def splitmix64(seed: int, k: int) -> int:
    """Draw k of the SplitMix64 sequence started at seed (reading A23)."""
    return int(_load().oracle_splitmix64(seed, k))


def skew_partition(rids: np.ndarray, n_src: int, num_runs: int, sample_size: int,
                   seed: int) -> np.ndarray:
    """Run boundaries from a sorted sample of the rids (section 2.3, P:466-475;
    S:162-170): uint32 [n_runs + 1], 0 < cuts < n_src strictly ascending."""
    rids = np.ascontiguousarray(rids, dtype=np.uint32)
    bounds = np.zeros(num_runs + 1, dtype=np.uint32)
    n = ctypes.c_uint64(0)
    if _load().oracle_skew_partition(_ptr(rids), rids.size, n_src, num_runs, sample_size, seed,
                                     _ptr(bounds), ctypes.byref(n)) != 0:
        raise ValueError("invalid argument")
    return bounds[:n.value + 1].copy()


def dpg_bounds(src: np.ndarray, rids: np.ndarray, bounds: np.ndarray):
    """Fig. 1 with runs [bounds[k], bounds[k+1]).  Returns a dict
    with ``dst``, ``run_start`` (n_runs + 1) and ``rid_pos`` (the positions of
    each run's entries, in Phase I order)."""
    src = _records(src)
    n_src, rec = src.shape
    rids = np.ascontiguousarray(rids, dtype=np.uint32)
    bounds = np.ascontiguousarray(bounds, dtype=np.uint32)
    n_runs = bounds.size - 1
    dst = np.zeros((rids.size, rec), dtype=np.uint8)
    run_start = np.zeros(n_runs + 1, dtype=np.uint64)
    rid_pos = np.zeros(rids.size, dtype=np.uint64)
    bad = ctypes.c_uint64(0)
    st = _load().oracle_dpg_bounds(_ptr(src), rec, n_src, _ptr(rids), rids.size, _ptr(bounds),
                                   n_runs, _ptr(dst), _ptr(run_start), _ptr(rid_pos),
                                   ctypes.byref(bad))
    _check(st, bad)
    return {"dst": dst, "run_start": run_start, "rid_pos": rid_pos}
