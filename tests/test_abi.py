"""Host-side tests of the C ABI (no GPU): the library loads, exports every
symbol include/dpg.h declares, validates arguments before touching CUDA, and
plans run lengths per the paper's constraints."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dpg():
    from tools.buildall import build_dpg
    build_dpg()
    import paper_cs_0308004_b200 as m
    return m


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "dpg.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dpg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(dpg):
    declared = _declared_symbols()
    assert "dpg_retrieve" in declared and "dpg_fk_join" in declared
    out = subprocess.check_output(["nm", "-D", "--defined-only", dpg.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(dpg.raw_lib(), s)
    assert set(dpg.EXPORTED) <= set(declared)


def test_library_is_sm100a_only(dpg):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dpg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", dpg.LIB_PATH],
                          capture_output=True, text=True).stdout
    # TMA bulk copies in the probe-gather kernel
    assert "UBLKCP" in sass


def test_status_strings(dpg):
    lib = dpg.raw_lib()
    assert lib.dpg_status_string(0) == b"DPG_OK"
    assert lib.dpg_status_string(2) == b"DPG_ERR_RID_RANGE"
    assert lib.dpg_version() >= 1


def test_argument_validation_before_any_cuda_call(dpg):
    lib = dpg.raw_lib()
    p = ctypes.c_void_p(0x10000)
    q = ctypes.c_void_p(0x90000000)
    r = ctypes.c_void_p(0x40000000)
    # rec == 0
    assert lib.dpg_retrieve(p, 0, 10, r, 10, q, None) == dpg.DPG_ERR_INVALID_ARG
    # n_out == 0: no-op
    assert lib.dpg_retrieve(None, 100, 10, None, 0, None, None) == dpg.DPG_OK
    # NULL pointer with nonzero count
    assert lib.dpg_retrieve(None, 100, 10, r, 10, q, None) == dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_retrieve(p, 100, 10, None, 10, q, None) == dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_retrieve(p, 100, 10, r, 10, None, None) == dpg.DPG_ERR_INVALID_ARG
    # n_src == 0 with n_out > 0
    assert lib.dpg_retrieve(p, 100, 0, r, 10, q, None) == dpg.DPG_ERR_INVALID_ARG
    # dst overlapping src (in-place is not the paper's problem)
    assert lib.dpg_retrieve(p, 100, 10, r, 10, ctypes.c_void_p(0x10000 + 500), None) == \
        dpg.DPG_ERR_INVALID_ARG
    # dst overlapping rids
    assert lib.dpg_retrieve(p, 4, 10, r, 10, r, None) == dpg.DPG_ERR_INVALID_ARG
    # n_out >= 2^32
    assert lib.dpg_retrieve(p, 1, 10, r, 1 << 32, q, None) == dpg.DPG_ERR_UNSUPPORTED
    # byte-size overflow
    assert lib.dpg_retrieve(p, 1 << 40, 1 << 30, r, 10, q, None) == dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_retrieve_direct(p, 0, 10, r, 10, q, None) == dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_fk_join(p, 16, 10, r, None, 64, 10, q, None) == dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_scatter_rows(p, 0, r, 10, q, 10, None) == dpg.DPG_ERR_INVALID_ARG


@pytest.mark.parametrize("rec,n,L,K,path", [
    (100, 65536, 128, 512, 1),        # config 1: runs shrink for load balance
    (100, 1048576, 512, 2048, 1),     # config 2: fused kernel, 4 stages of 50 KB runs
    (64, 16777216, 512, 32768, 1),    # config 3 at rec 64: smaller Phase I tiles
    (256, 16777216, 256, 65536, 2),   # too many runs for the fused kernel
])
def test_plan_run_length(dpg, rec, n, L, K, path):
    """Shared-memory runs (paths 1 and 2): the plan when the source exceeds the
    L2 budget, or on request."""
    p = dpg.dpg_plan(rec, n, n, 0, 148, path=path)
    assert p["run_len"] == L and p["num_runs"] == K and p["path"] == path
    assert p["run_len"] & (p["run_len"] - 1) == 0            # power of two
    assert p["smem_bytes"] <= 232448                          # two stages fit one SM
    assert p["slot_pairs"] >= p["run_len"]                    # a permutation's run fits one stage
    assert p["run_len"] * rec <= (p["smem_bytes"] - 128) // p["nstages"]
    m = dpg.dpg_plan(rec, n, n, 0, 148, path=2)
    assert m["path"] == 2 and m["nstages"] == 2
    # Phase I: shared-memory histograms while K counters fit, else radix
    # passes of 8 bits over the run index (8-byte elements carrying the rid)
    if m["num_runs"] > 24576 or n >= 4 << 20:
        assert m["dist_radix"] == (int(m["num_runs"] - 1).bit_length() + 7) // 8
        assert m["pair_bytes"] == 8 and m["grid_distribute"] == 3 * 148
    else:
        assert m["dist_radix"] == 0
    r = dpg.dpg_plan(rec, n, n, 0, 148, path=2, hist_mode=3)
    assert r["dist_radix"] >= 1 and r["pair_bytes"] == 8


@pytest.mark.parametrize("rec,n,auto_path", [
    (100, 65536, 3),                  # config 1: 6.6 MB source, one L2 run
    (100, 1048576, 3),                # config 2: 105 MB source <= 7/8 of the L2, one staged run
    (64, 16777216, 1),                # config 3 at rec 64: 1.07 GB, shared-memory runs
    (8, 1 << 24, 6),                  # 134 MB source > budget, small records: three sequential passes
    (32, 1 << 24, 6),
])
def test_plan_l2_run_rule(dpg, rec, n, auto_path):
    """The run is sized to the cache: one run (path 3) when the
    whole source fits the L2 budget (7/8 of 126 MB with no device), else
    shared-memory runs: for records up to 32 bytes the three sequential passes
    (path 6), else the fused / multi-kernel plans."""
    run_budget = (126 << 20) // 16 * 7                 # one L2 run (measured retention)
    p = dpg.dpg_plan(rec, n, n, 0, 148)
    assert p["path"] == auto_path
    q = dpg.dpg_plan(rec, n, n, 0, 148, path=4) if rec % 4 == 0 and rec <= 116 and n <= 1 << 20 else None
    if q is not None:                                  # two L2 runs on request
        assert q["num_runs"] == 2 and 2 * q["run_len"] >= n
    if p["path"] == 3:
        assert p["num_runs"] == 1 and p["run_len"] >= n
    if p["path"] == 4:
        assert p["num_runs"] == 2 and p["run_len"] * rec <= run_budget < n * rec
        assert p["run_len"] & (p["run_len"] - 1) == 0 and 2 * p["run_len"] >= n


def test_plan_pair_packing_and_overrides(dpg):
    c2 = dpg.dpg_plan(100, 1 << 20, 1 << 20, path=1)
    assert c2["gather"] == 2 and c2["pair_bytes"] == 2                # rows straddle sectors
    c2 = dpg.dpg_plan(100, 1 << 20, 1 << 20, path=1, gather=1)
    assert c2["gather"] == 1 and c2["pair_bytes"] == 4                # 9 + 20 bits packed
    assert c2["slot_pairs"] == 672                                    # CAP = L + L/4 + 32
    assert dpg.dpg_plan(100, 1 << 20, 1 << 20, gather=2)["pair_bytes"] == 2   # u16 locals
    assert dpg.dpg_plan(128, 1 << 20, 1 << 20, path=1)["gather"] == 1  # whole sectors
    assert dpg.dpg_plan(64, 1 << 24, 1 << 26)["pair_bytes"] == 8      # 10 + 26 bits
    assert dpg.dpg_plan(100, 1 << 20, 1 << 20, pair_bytes=8, gather=1)["pair_bytes"] == 8
    assert dpg.dpg_plan(100, 1 << 20, 1 << 20, pair_bytes=8, gather=2)["pair_bytes"] == 4
    p = dpg.dpg_plan(3, 12, 12, log2_run=2)
    assert p["run_len"] == 4 and p["num_runs"] == 3                   # Fig. 2 geometry
    assert dpg.dpg_plan(64, 1 << 24, 1 << 26, path=2)["path"] == 2
    with pytest.raises(dpg.DPGError):                                 # payload: multi-kernel only
        dpg.dpg_plan(64, 1 << 24, 1 << 26, pay_bytes=16, path=1)
    with pytest.raises(dpg.DPGError):
        dpg.dpg_plan(0, 10, 10)
    j = dpg.dpg_plan(64, 1 << 24, 1 << 26, pay_bytes=16)
    assert j["pay_bytes"] == 16 and j["word_bytes"] == 16


def test_bounds_entry_points_host_checks(dpg):
    """Boundary-mode runs (section 2.3): host-side validation and the merged
    layout's size (bounds merged with the multiples of L), no CUDA call."""
    lib = dpg.raw_lib()
    U32 = ctypes.c_uint32
    p = ctypes.c_void_p(0x10000)
    q = ctypes.c_void_p(0x90000000)
    r = ctypes.c_void_p(0x40000000)
    K = ctypes.c_uint64(0)

    def b(*v):
        return (U32 * len(v))(*v)

    # size query: K = n_runs + ceil(n_src / L) - 1
    assert lib.dpg_distribute_bounds(None, 0, 1000, b(0, 10, 500, 1000), 3, 8, None, None,
                                     ctypes.byref(K), None) == dpg.DPG_OK
    assert K.value == 3 + 4 - 1
    assert lib.dpg_distribute_bounds(None, 0, 100, b(0, 100), 1, 10, None, None,
                                     ctypes.byref(K), None) == dpg.DPG_OK
    assert K.value == 1
    for bad in [b(1, 100), b(0, 99), b(0, 60, 50, 100)]:
        n = len(bad) - 1
        assert lib.dpg_distribute_bounds(None, 0, 100, bad, n, 4, None, None, ctypes.byref(K),
                                         None) == dpg.DPG_ERR_INVALID_ARG
        assert lib.dpg_retrieve_bounds(p, 8, 100, r, 10, bad, n, q, None) == \
            dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_retrieve_bounds(p, 8, 100, r, 10, None, 1, q, None) == dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_retrieve_bounds(p, 0, 100, r, 10, b(0, 100), 1, q, None) == \
        dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_retrieve_bounds(p, 8, 100, r, 0, b(0, 100), 1, q, None) == dpg.DPG_OK
    n_runs = U32(0)
    out = (U32 * 10)()
    assert lib.dpg_skew_partition(r, 0, 100, 4, 16, 0, out, ctypes.byref(n_runs), None) == \
        dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_skew_partition(r, 10, 100, 8, 4, 0, out, ctypes.byref(n_runs), None) == \
        dpg.DPG_ERR_INVALID_ARG
    assert lib.dpg_skew_partition(r, 10, 100, 4, 40000, 0, out, ctypes.byref(n_runs), None) == \
        dpg.DPG_ERR_UNSUPPORTED


def test_library_has_no_undefined_internal_symbols(dpg):
    """Every internal (namespace dpg) function the translation units call is
    defined in the library: an undefined one would only fail at dlopen on the
    GPU box."""
    out = subprocess.check_output(["nm", "-D", "--undefined-only", dpg.LIB_PATH], text=True)
    missing = [line.split()[-1] for line in out.splitlines() if "_ZN3dpg" in line]
    assert not missing, missing


def test_host_entries_validate_before_cuda(dpg):
    lib = dpg.raw_lib()
    p = ctypes.c_void_p(0x10000)
    for fn in (lib.dpg_retrieve_host, lib.dpg_retrieve_host_async):
        assert fn(p, 0, 10, p, 10, p, None) == dpg.DPG_ERR_INVALID_ARG      # rec == 0
        assert fn(p, 8, 10, p, 0, p, None) == dpg.DPG_OK                    # nothing to do
        assert fn(None, 8, 10, p, 10, p, None) == dpg.DPG_ERR_INVALID_ARG
        assert fn(p, 8, 0, p, 10, p, None) == dpg.DPG_ERR_INVALID_ARG       # n_src == 0
        assert fn(p, 1 << 40, 1 << 30, p, 10, p, None) == dpg.DPG_ERR_INVALID_ARG   # overflow


def test_fuzz_cases_reach_every_plan(dpg):
    """The randomised GPU parity cases (test_gpu_fuzz.py) are only worth
    their run time if every forced plan accepts some of them and the
    automatic planner picks more than one path: checked here with the host
    planner."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import test_gpu_fuzz as fz
    ran = {name: 0 for name, _ in fz.VARIANTS}
    auto = set()
    for (_, rec, _, n_src, n_out, _) in fz._cases():
        for name, o in fz.VARIANTS:
            try:
                p = dpg.dpg_plan(rec, n_src, n_out, **fz._opts(name, o, n_src))
            except dpg.DPGError:
                continue
            ran[name] += 1
            if name == "auto":
                auto.add(p["path"])
    assert min(ran.values()) >= 10, ran
    assert {1, 3, 6} <= auto, auto


@pytest.mark.parametrize("rec,n", [(4, 1 << 24), (4, 1 << 26), (8, 1 << 24), (16, 1 << 24), (8, 1 << 26)])
def test_plan_seq3_phase1_occupancy(dpg, rec, n):
    """Path 6's tile: Phase III's buffer bounds it; where one Phase I CTA
    (T rids + T 16-bit offsets + two K+1 count columns, seq3.cu) would fill an
    SM's 228 KB, the tile shrinks by at most 20 % so that two share it
    (profiles/r02_s3_p6dist.md)."""
    p = dpg.dpg_plan(rec, n, n, 0, 148)
    assert p["path"] == 6
    T, K = p["tile"], p["num_runs"]
    assert T % 16 == 0
    smem = 256 + 4 * T + ((2 * T + 15) & ~15) + 2 * ((K + 1) * 4 + 16)
    per_sm = 233472 // (smem + 1024)
    assert per_sm >= 1 and p["grid_distribute"] == min(-(-n // T), min(4, per_sm) * 148)
    if rec == 4:                                  # 117 KB at the buffer's tile: shrunk to two per SM
        assert per_sm == 2
        full = min(32768, (110 << 10) // (rec + 2)) & ~15
        assert 0.8 * full <= T < full
