"""B200-native DPG record retrieval (arXiv cs/0308004) -- Python binding.

A thin ctypes layer over ``libdpg.so`` (C ABI declared in ``include/dpg.h``):
argument marshalling only.  Every step of the path runs in the library's
CUDA kernels; PyTorch supplies device memory and the current stream.  There
is no CPU fallback: importing this package raises if ``libdpg.so`` has not
been built (``python -m paper_cs_0308004_b200.build``).

Functions carry the C ABI's names:

* :func:`dpg_retrieve`        ``dst[i] = src[rids[i]]`` by distribute-probe-gather (Fig. 1)
* :func:`dpg_sort`            three-phase key-pointer sort with DPG as phase 3
* :func:`dpg_retrieve_direct` the standard direct retrieval, the measured comparison
* :func:`dpg_fk_join`         DPG-Move join rows ``fact[i] ++ dim[fk[i]]``
* :func:`dpg_distribute`      Phase I alone, for tests
* :func:`dpg_scatter_rows`    ``dst[pos[k]] = rows[k]`` (multi-GPU reply scatter)
* :func:`dpg_retrieve_host`   end-to-end entry with host buffers
* :func:`dpg_plan`            the host-side plan (run length L, stages, grids)
* :func:`dpg_sync_status`     device-side rid-range errors
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdpg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_cs_0308004_b200.build` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

DPG_OK, DPG_ERR_INVALID_ARG, DPG_ERR_RID_RANGE, DPG_ERR_UNSUPPORTED, DPG_ERR_OOM, \
    DPG_ERR_CUDA, DPG_ERR_NCCL = range(7)

EXPORTED = (
    "dpg_plan", "dpg_retrieve", "dpg_retrieve_ex", "dpg_retrieve_direct", "dpg_fk_join",
    "dpg_fk_join_ex", "dpg_distribute", "dpg_scatter_rows", "dpg_retrieve_host",
    "dpg_release_cache", "dpg_sync_status", "dpg_status_string", "dpg_last_launch_count",
    "dpg_version", "dpg_phase_timing", "dpg_phase_times", "dpg_debug_phase_stamps",
    "dpg_retrieve_direct_ex", "dpg_l2_prefetch", "dpg_partition", "dpg_last_path",
    "dpg_phase_times_ex", "dpg_retrieve_dist_loopback", "dpg_fk_join_direct",
    "dpg_skew_partition", "dpg_retrieve_bounds", "dpg_distribute_bounds",
    "dpg_retrieve_host_async", "dpg_exchange_plan",
)


class DPGError(RuntimeError):
    def __init__(self, status: int, where: str, index: int | None = None):
        name = _lib.dpg_status_string(status).decode()
        msg = f"{where}: {name}" + (f" at position {index}" if index is not None else "")
        super().__init__(msg)
        self.status = status
        self.index = index


class Plan(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("log2_run", "pair_bytes")] + [
        ("run_len", ctypes.c_uint64), ("num_runs", ctypes.c_uint64)] + [
        (n, ctypes.c_uint32) for n in ("word_bytes", "slot_pairs", "smem_bytes",
                                       "grid_distribute", "grid_probe", "hist_in_smem",
                                       "pay_bytes", "path", "nstages", "stage_bytes",
                                       "gather", "npre", "rid_cache", "hist_warps",
                                       "tile", "cluster", "dist_radix")]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class Options(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("log2_run", "grid_distribute", "grid_probe",
                                               "pair_bytes", "hist_mode", "path", "gather",
                                               "cluster")]


_P, _U, _S, _I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_int
_st = ctypes.c_int
_sigs = {
    "dpg_plan": [_S, _U, _U, _S, _P, _I, _P],
    "dpg_retrieve": [_P, _S, _U, _P, _U, _P, _P],
    "dpg_retrieve_ex": [_P, _S, _U, _P, _U, _P, _P, _P],
    "dpg_retrieve_direct": [_P, _S, _U, _P, _U, _P, _P],
    "dpg_fk_join": [_P, _S, _U, _P, _P, _S, _U, _P, _P],
    "dpg_fk_join_ex": [_P, _S, _U, _P, _P, _S, _U, _P, _P, _P],
    "dpg_distribute": [_P, _U, _U, ctypes.c_uint32, _P, _P, _P, _P],
    "dpg_scatter_rows": [_P, _S, _P, _U, _P, _U, _P],
    "dpg_retrieve_host": [_P, _S, _U, _P, _U, _P, _P],
    "dpg_retrieve_host_async": [_P, _S, _U, _P, _U, _P, _P],
    "dpg_exchange_plan": [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P],
    "dpg_sync_status": [_P, _P],
    "dpg_retrieve_direct_ex": [_P, _S, _U, _P, _U, _P, _P, _I],
    "dpg_l2_prefetch": [_P, _U, _P],
    "dpg_partition": [_P, ctypes.c_uint32, _U, _U, ctypes.c_uint32, ctypes.c_uint32, _P, _P, _P,
                      _P],
    "dpg_sort_rids": [_P, _S, _U, _S, _S, _P, _P],
    "dpg_partition_inv": [_P, ctypes.c_uint32, _U, _U, ctypes.c_uint32, ctypes.c_uint32, _P, _P,
                          _P, _P],
    "dpg_gather_rows": [_P, _S, _U, _P, _U, _P, _P],
    "dpg_sort": [_P, _S, _U, _S, _S, _P, _P],
    "dpg_fk_join_sort": [_P, _S, _U, _P, _P, _S, _U, _P, _P],
    "dpg_fk_join_direct": [_P, _S, _U, _P, _P, _S, _U, _P, _P],
    "dpg_retrieve_segments": [_P, _S, _U, _P, _U, ctypes.c_uint32, _P, _P, _P],
    "dpg_ipc_alloc": [_S, _P, _P],
    "dpg_get_unique_id": [_P],
    "dpg_hash_lookup": [_P, ctypes.c_uint32, _P, _P, _U, _P, _P, ctypes.c_uint32],
    "dpg_hash_lookup_direct": [_P, ctypes.c_uint32, _P, _P, _U, _P, _P],
    "dpg_btree_lookup": [_P, _P, ctypes.c_uint32, _P, _P, _U, _P, _P, ctypes.c_uint32],
    "dpg_btree_lookup_direct": [_P, _P, ctypes.c_uint32, _P, _P, _U, _P, _P],
    "dpg_comm_create": [_P, ctypes.c_int, ctypes.c_int, _P],
    "dpg_retrieve_dist": [_P, _P, _S, _U, _P, _U, _P, _P],
    "dpg_retrieve_dist_loopback": [ctypes.c_int, _P, _S, _U, _P, _P, _P, _P],
    "dpg_comm_destroy": [_P],
    "dpg_ipc_open": [_P, _P],
    "dpg_ipc_close": [_P],
    "dpg_ipc_free": [_P],
    "dpg_skew_partition": [_P, _U, _U, ctypes.c_uint32, ctypes.c_uint32, _U, _P, _P, _P],
    "dpg_retrieve_bounds": [_P, _S, _U, _P, _U, _P, _U, _P, _P],
    "dpg_distribute_bounds": [_P, _U, _U, _P, _U, ctypes.c_uint32, _P, _P, _P, _P],
}
for _name, _args in _sigs.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _st
_lib.dpg_status_string.argtypes = [_st]
_lib.dpg_status_string.restype = ctypes.c_char_p
_lib.dpg_last_launch_count.restype = ctypes.c_uint32
_lib.dpg_last_path.restype = ctypes.c_uint32
_lib.dpg_version.restype = ctypes.c_int
_lib.dpg_release_cache.restype = None
_lib.dpg_phase_timing.argtypes = [ctypes.c_int]
_lib.dpg_phase_timing.restype = None
_lib.dpg_phase_times.argtypes = [_P, _P, _P]
_lib.dpg_phase_times.restype = _st
_lib.dpg_phase_times_ex.argtypes = [_P, _P, _P, _P]
_lib.dpg_phase_times_ex.restype = _st


def _check(status: int, where: str):
    if status != DPG_OK:
        raise DPGError(status, where)


def _options(**kw) -> Options | None:
    if not kw or all(v in (None, 0) for v in kw.values()):
        return None
    o = Options()
    for k, v in kw.items():
        if v:
            setattr(o, k, int(v))
    return o


def _ref(o):
    return None if o is None else ctypes.byref(o)


def dpg_plan(rec_bytes: int, n_src: int, n_out: int, pay_bytes: int = 0, sm_count: int = 148,
             **opts) -> dict:
    """The plan the library would choose (host-only; no GPU needed)."""
    p = Plan()
    _check(_lib.dpg_plan(rec_bytes, n_src, n_out, pay_bytes, _ref(_options(**opts)), sm_count,
                         ctypes.byref(p)), "dpg_plan")
    return p.as_dict()


def last_launch_count() -> int:
    return int(_lib.dpg_last_launch_count())


def last_path() -> int:
    """Plan path the last dpg_retrieve / dpg_fk_join on this thread ran (after
    the data skew check)."""
    return int(_lib.dpg_last_path())


def dpg_phase_timing(enable: bool = True):
    """Record CUDA events around Phase I and the probe-gather kernel of every
    call (on the call's stream) until disabled."""
    _lib.dpg_phase_timing(1 if enable else 0)


def dpg_phase_times() -> tuple[float, float, int]:
    """(distribute_ms, probe_gather_ms, calls) summed since the last read."""
    d, p, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
    _check(_lib.dpg_phase_times(ctypes.byref(d), ctypes.byref(p), ctypes.byref(c)),
           "dpg_phase_times")
    return d.value, p.value, c.value


def dpg_phase_times_ex() -> tuple[float, float, float, int]:
    """(phase1_ms, phase2_ms, phase3_ms, calls) summed since the last read;
    phase3_ms is nonzero only for the three-kernel plan (path 6), whose Phase
    II and Phase III are timed separately (else phase2_ms covers both)."""
    a, b, c, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
    _check(_lib.dpg_phase_times_ex(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                   ctypes.byref(n)), "dpg_phase_times_ex")
    return a.value, b.value, c.value, n.value


# ---------------------------------------------------------------------------
# torch-facing wrappers (device tensors; stream = torch's current stream)
# ---------------------------------------------------------------------------
def _torch():
    import torch
    return torch


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _records(t, name):
    torch = _torch()
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.uint8:
        raise ValueError(f"{name} must be uint8 [n, rec_bytes]")
    if t.dim() == 1:
        t = t.view(-1, 1)
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _rid_tensor(t, name="rids"):
    torch = _torch()
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype not in (torch.int32, torch.uint32):
        raise ValueError(f"{name} must be int32/uint32 (read as uint32)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def dpg_retrieve(src, rids, dst=None, stream=None, log2_run=0, grid_distribute=0, grid_probe=0,
                 pair_bytes=0, hist_mode=0, path=0, gather=0, cluster=0):
    """``dst[i] = src[rids[i]]`` by DPG.  src: uint8 CUDA [n_src, rec]; rids:
    int32/uint32 CUDA [n_out].  Returns dst (uint8 [n_out, rec])."""
    torch = _torch()
    src = _records(src, "src")
    rids = _rid_tensor(rids)
    n_src, rec = src.shape
    n_out = rids.numel()
    if dst is None:
        dst = torch.empty((n_out, rec), dtype=torch.uint8, device=src.device)
    o = _options(log2_run=log2_run, grid_distribute=grid_distribute, grid_probe=grid_probe,
                 pair_bytes=pair_bytes, hist_mode=hist_mode, path=path, gather=gather,
                 cluster=cluster)
    _check(_lib.dpg_retrieve_ex(src.data_ptr(), rec, n_src, rids.data_ptr(), n_out,
                                dst.data_ptr(), _stream_ptr(stream), _ref(o)), "dpg_retrieve")
    return dst


def dpg_retrieve_direct(src, rids, dst=None, stream=None):
    """The paper's standard direct retrieval on the GPU."""
    torch = _torch()
    src = _records(src, "src")
    rids = _rid_tensor(rids)
    n_src, rec = src.shape
    n_out = rids.numel()
    if dst is None:
        dst = torch.empty((n_out, rec), dtype=torch.uint8, device=src.device)
    _check(_lib.dpg_retrieve_direct(src.data_ptr(), rec, n_src, rids.data_ptr(), n_out,
                                    dst.data_ptr(), _stream_ptr(stream)), "dpg_retrieve_direct")
    return dst


def dpg_retrieve_direct_ex(src, rids, dst=None, stream=None, hint=0):
    """Direct retrieval with L2 hints (0 plain, 1 stream, 2 L2-resident source)."""
    torch = _torch()
    src = _records(src, "src")
    rids = _rid_tensor(rids)
    n_src, rec = src.shape
    n_out = rids.numel()
    if dst is None:
        dst = torch.empty((n_out, rec), dtype=torch.uint8, device=src.device)
    _check(_lib.dpg_retrieve_direct_ex(src.data_ptr(), rec, n_src, rids.data_ptr(), n_out,
                                       dst.data_ptr(), _stream_ptr(stream), hint),
           "dpg_retrieve_direct_ex")
    return dst


def dpg_l2_prefetch(t, stream=None):
    """Stage tensor t's bytes into L2 (evict_last)."""
    _check(_lib.dpg_l2_prefetch(t.data_ptr(), t.numel() * t.element_size(), _stream_ptr(stream)),
           "dpg_l2_prefetch")


def dpg_fk_join(fact, fk_col, dim, out=None, stream=None, **opts):
    """DPG-Move join: out row i = fact[i] ++ dim[fk_col[i]]."""
    torch = _torch()
    fact = _records(fact, "fact")
    dim = _records(dim, "dim")
    fk_col = _rid_tensor(fk_col, "fk_col")
    n_fact, fact_bytes = fact.shape
    n_dim, rec = dim.shape
    if fk_col.numel() != n_fact:
        raise ValueError("fk_col must have one entry per fact row")
    if out is None:
        out = torch.empty((n_fact, fact_bytes + rec), dtype=torch.uint8, device=dim.device)
    _check(_lib.dpg_fk_join_ex(fact.data_ptr(), fact_bytes, n_fact, fk_col.data_ptr(),
                               dim.data_ptr(), rec, n_dim, out.data_ptr(), _stream_ptr(stream),
                               _ref(_options(**opts))), "dpg_fk_join")
    return out


def dpg_fk_join_direct(fact, fk_col, dim, out=None, stream=None):
    """The direct join (one random dim access per fact row), same rows as
    dpg_fk_join: the measured comparison."""
    torch = _torch()
    fact = _records(fact, "fact")
    dim = _records(dim, "dim")
    fk_col = _rid_tensor(fk_col, "fk_col")
    n_fact, fact_bytes = fact.shape
    n_dim, rec = dim.shape
    if out is None:
        out = torch.empty((n_fact, fact_bytes + rec), dtype=torch.uint8, device=dim.device)
    _check(_lib.dpg_fk_join_direct(fact.data_ptr(), fact_bytes, n_fact, fk_col.data_ptr(),
                                   dim.data_ptr(), rec, n_dim, out.data_ptr(), _stream_ptr(stream)),
           "dpg_fk_join_direct")
    return out


def dpg_distribute(rids, n_src: int, log2_run: int, stream=None, **opts):
    """Phase I alone.  Returns (pairs uint64 [n_out] = local | pos << 32,
    run_start uint64 [K+1]) as int64 CUDA tensors."""
    torch = _torch()
    rids = _rid_tensor(rids)
    n_out = rids.numel()
    K = (n_src + (1 << log2_run) - 1) >> log2_run
    pairs = torch.empty(max(n_out, 1), dtype=torch.int64, device=rids.device)
    rs = torch.empty(K + 1, dtype=torch.int64, device=rids.device)
    _check(_lib.dpg_distribute(rids.data_ptr(), n_out, n_src, log2_run, pairs.data_ptr(),
                               rs.data_ptr(), _stream_ptr(stream), _ref(_options(**opts))),
           "dpg_distribute")
    return pairs[:n_out], rs


def _host_bounds(bounds):
    import numpy as np
    b = np.ascontiguousarray(np.asarray(bounds), dtype=np.uint32)
    if b.ndim != 1 or b.size < 2:
        raise ValueError("bounds: 1-D, at least two entries (0 ... n_src)")
    return b


def dpg_skew_partition(rids, n_src: int, num_runs: int, sample_size: int = 16384, seed: int = 0,
                       stream=None):
    """Run boundaries from a sorted sample of the rids (section 2.3):
    numpy uint32 [n_runs + 1] = 0, cuts..., n_src (synchronous)."""
    import numpy as np
    rids = _rid_tensor(rids)
    out = np.zeros(num_runs + 1, dtype=np.uint32)
    n = ctypes.c_uint32(0)
    _check(_lib.dpg_skew_partition(rids.data_ptr(), rids.numel(), n_src, num_runs, sample_size,
                                   seed, out.ctypes.data, ctypes.addressof(n),
                                   _stream_ptr(stream)), "dpg_skew_partition")
    return out[:n.value + 1].copy()


def dpg_retrieve_bounds(src, rids, bounds, dst=None, stream=None):
    """``dst[i] = src[rids[i]]`` by DPG with runs [bounds[k], bounds[k+1])
    (host array; bounds[0] = 0, bounds[-1] = n_src)."""
    torch = _torch()
    src = _records(src, "src")
    rids = _rid_tensor(rids)
    n_src, rec = src.shape
    n_out = rids.numel()
    b = _host_bounds(bounds)
    if dst is None:
        dst = torch.empty((n_out, rec), dtype=torch.uint8, device=src.device)
    _check(_lib.dpg_retrieve_bounds(src.data_ptr(), rec, n_src, rids.data_ptr(), n_out,
                                    b.ctypes.data, b.size - 1, dst.data_ptr(),
                                    _stream_ptr(stream)), "dpg_retrieve_bounds")
    return dst


def dpg_distribute_bounds(rids, n_src: int, bounds, log2_run: int, stream=None):
    """Phase I over the bounds merged with the multiples of 2^log2_run.
    Returns (pairs int64 [n_out] = (rid - run start) | pos << 32, run_start
    int64 [K+1]) as CUDA tensors."""
    torch = _torch()
    rids = _rid_tensor(rids)
    n_out = rids.numel()
    b = _host_bounds(bounds)
    K = ctypes.c_uint64(0)
    _check(_lib.dpg_distribute_bounds(None, n_out, n_src, b.ctypes.data, b.size - 1, log2_run,
                                      None, None, ctypes.addressof(K), None),
           "dpg_distribute_bounds")
    pairs = torch.empty(max(n_out, 1), dtype=torch.int64, device=rids.device)
    rs = torch.empty(K.value + 1, dtype=torch.int64, device=rids.device)
    _check(_lib.dpg_distribute_bounds(rids.data_ptr(), n_out, n_src, b.ctypes.data, b.size - 1,
                                      log2_run, pairs.data_ptr(), rs.data_ptr(),
                                      ctypes.addressof(K), _stream_ptr(stream)),
           "dpg_distribute_bounds")
    return pairs[:n_out], rs


def dpg_exchange_plan(counts, me: int) -> dict:
    """The multi-GPU exchange's offsets for rank `me` from the P x (P+1) count
    matrix (host, no GPU): roff, soff (P+1 each), win_row (P), n_req, cap."""
    import numpy as np
    C = np.ascontiguousarray(np.asarray(counts), dtype=np.uint64)
    P = C.shape[0]
    if C.shape != (P, P + 1):
        raise ValueError("counts must be P x (P + 1)")
    roff = np.zeros(P + 1, np.uint64)
    soff = np.zeros(P + 1, np.uint64)
    win = np.zeros(P, np.uint64)
    n_req, cap = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(_lib.dpg_exchange_plan(C.ctypes.data, P, me, roff.ctypes.data, soff.ctypes.data,
                                  win.ctypes.data, ctypes.addressof(n_req), ctypes.addressof(cap)),
           "dpg_exchange_plan")
    return {"roff": roff, "soff": soff, "win_row": win, "n_req": n_req.value, "cap": cap.value}


def dpg_partition(rids, n_src_total: int, log2_span: int, parts: int, stream=None):
    """Distribute rids (CUDA int32/uint32/int64/uint64) to owners rid >> log2_span.
    Returns (local int32 [m], pos int32 [m], counts int64 [parts]) as CUDA
    tensors, grouped by owner (m = number of valid rids)."""
    torch = _torch()
    if not rids.is_cuda or not rids.is_contiguous():
        raise ValueError("rids must be a contiguous CUDA tensor (no CPU fallback)")
    rb = rids.element_size()
    if rb not in (4, 8):
        raise ValueError("rids must be 32- or 64-bit")
    n = rids.numel()
    local = torch.empty(max(n, 1), dtype=torch.int32, device=rids.device)
    pos = torch.empty(max(n, 1), dtype=torch.int32, device=rids.device)
    counts = torch.empty(parts, dtype=torch.int64, device=rids.device)
    _check(_lib.dpg_partition(rids.data_ptr(), rb, n, n_src_total, log2_span, parts,
                              local.data_ptr(), pos.data_ptr(), counts.data_ptr(),
                              _stream_ptr(stream)), "dpg_partition")
    return local, pos, counts


def dpg_partition_inv(rids, n_src_total: int, log2_span: int, parts: int, stream=None):
    """Group rids (CUDA, 32/64-bit) by owner rid >> log2_span.  Returns (local
    int32 [n], inv int32 [n], counts int64 [parts]): the owner-local offsets
    owner by owner (the first sum(counts) entries), and for every row the
    position of its request (-1 for a rid out of range)."""
    torch = _torch()
    if not rids.is_cuda or not rids.is_contiguous():
        raise ValueError("rids must be a contiguous CUDA tensor (no CPU fallback)")
    rb = rids.element_size()
    if rb not in (4, 8):
        raise ValueError("rids must be 32- or 64-bit")
    n = rids.numel()
    local = torch.empty(max(n, 1), dtype=torch.int32, device=rids.device)
    inv = torch.empty(max(n, 1), dtype=torch.int32, device=rids.device)
    counts = torch.empty(parts, dtype=torch.int64, device=rids.device)
    _check(_lib.dpg_partition_inv(rids.data_ptr(), rb, n, n_src_total, log2_span, parts,
                                  local.data_ptr(), inv.data_ptr(), counts.data_ptr(),
                                  _stream_ptr(stream)), "dpg_partition_inv")
    return local, inv[:n], counts


def dpg_gather_rows(rows, inv, dst, stream=None, n_rows=None):
    """dst[i] = rows[inv[i]] for inv[i] in range (other rows left unwritten).
    rows: a uint8 [n_rows, rec] CUDA tensor, or an integer device address of
    n_rows rows of dst's row size (a receive window)."""
    inv = _rid_tensor(inv, "inv")
    dst = _records(dst, "dst")
    rec = dst.shape[1]
    if isinstance(rows, int):
        ptr = rows
    else:
        rows = _records(rows, "rows")
        n_rows, rec = rows.shape
        ptr = rows.data_ptr()
    _check(_lib.dpg_gather_rows(ptr, rec, n_rows, inv.data_ptr(), inv.numel(),
                                dst.data_ptr(), _stream_ptr(stream)), "dpg_gather_rows")
    return dst


def dpg_scatter_rows(rows, pos, dst, stream=None):
    """dst[pos[k]] = rows[k] (pos distinct, uint32)."""
    rows = _records(rows, "rows")
    pos = _rid_tensor(pos, "pos")
    dst = _records(dst, "dst")
    n, rec = rows.shape
    _check(_lib.dpg_scatter_rows(rows.data_ptr(), rec, pos.data_ptr(), n, dst.data_ptr(),
                                 dst.shape[0], _stream_ptr(stream)), "dpg_scatter_rows")
    return dst


def dpg_retrieve_host(src, rids, dst, stream=None, synchronize=True):
    """End-to-end retrieval with HOST tensors (pinned for full PCIe speed):
    H2D of src and rids, DPG on the GPU, D2H of dst, synchronise.  With
    synchronize=False (dpg_retrieve_host_async) the work is only enqueued on
    `stream`; dst is complete once the stream is synchronised."""
    for t, n in ((src, "src"), (rids, "rids"), (dst, "dst")):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{n} must be a contiguous host tensor")
    n_src, rec = src.shape
    fn = _lib.dpg_retrieve_host if synchronize else _lib.dpg_retrieve_host_async
    _check(fn(src.data_ptr(), rec, n_src, rids.data_ptr(), rids.numel(), dst.data_ptr(),
              _stream_ptr(stream)), "dpg_retrieve_host")
    return dst


def dpg_retrieve_segments(src, rids, seg_rows, seg_dst, stream=None):
    """D[k] = src[rids[k]] with the output split into segments: the rows of
    segment q go to seg_dst[q] (a uint8 CUDA tensor, or an integer device
    address such as a peer window from ipc_open) in order."""
    src = _records(src, "src")
    rids = _rid_tensor(rids, "rids")
    n_src, rec = src.shape
    nseg = len(seg_rows)
    if nseg != len(seg_dst):
        raise ValueError("seg_rows and seg_dst differ in length")
    rows = (ctypes.c_uint64 * nseg)(*[int(x) for x in seg_rows])
    ptrs = (ctypes.c_void_p * nseg)(*[int(d) if isinstance(d, int) else d.data_ptr()
                                      for d in seg_dst])
    _check(_lib.dpg_retrieve_segments(src.data_ptr(), rec, n_src, rids.data_ptr(), rids.numel(),
                                      nseg, ctypes.cast(rows, ctypes.c_void_p),
                                      ctypes.cast(ptrs, ctypes.c_void_p), _stream_ptr(stream)),
           "dpg_retrieve_segments")


def dpg_hash_lookup(table, pool, keys, out=None, stream=None, direct=False, log2_run=0):
    """Batch lookup: out[i] = rid of keys[i] in the hash index
    (table: uint32 [2^m, 4] CUDA tensor, pool: uint32 [P, 4]), 0xFFFFFFFF
    if absent.  direct=True: one random slot read per key instead of DPG."""
    torch = _torch()
    m = int(table.shape[0]).bit_length() - 1
    if table.shape[0] != 1 << m or table.shape[-1] != 4 or not table.is_cuda:
        raise ValueError("table must be a CUDA [2^m, 4] uint32/int32 tensor")
    keys = _rid_tensor(keys, "keys")
    if out is None:
        out = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
    if direct:
        _check(_lib.dpg_hash_lookup_direct(table.data_ptr(), m, pool.data_ptr(), keys.data_ptr(),
                                           keys.numel(), out.data_ptr(), _stream_ptr(stream)),
               "dpg_hash_lookup_direct")
    else:
        _check(_lib.dpg_hash_lookup(table.data_ptr(), m, pool.data_ptr(), keys.data_ptr(),
                                    keys.numel(), out.data_ptr(), _stream_ptr(stream), log2_run),
               "dpg_hash_lookup")
    return out


def btree_to_device(levels, rids, device="cuda"):
    """The B+-tree levels (numpy uint32 arrays, level 0 = sorted keys) and the
    rids as CUDA tensors, each level padded to a multiple of 16 entries."""
    torch = _torch()
    out = []
    for lv in levels:
        pad = (-lv.size) % 16
        a = np.concatenate([lv, np.full(pad, 0xFFFFFFFF, dtype=np.uint32)]) if pad else lv
        out.append(torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).to(device))
    r = torch.from_numpy(np.ascontiguousarray(rids, dtype=np.uint32).view(np.int32)).to(device)
    return out, [int(lv.size) for lv in levels], r


def dpg_btree_lookup(levels, level_n, rids, keys, out=None, stream=None, direct=False, log2_run=0):
    """Batch lookup in an enhanced B+-tree: out[i] = rid of
    keys[i], 0xFFFFFFFF if absent.  levels/level_n/rids from btree_to_device."""
    torch = _torch()
    keys = _rid_tensor(keys, "keys")
    if out is None:
        out = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
    L = len(levels)
    ptrs = (ctypes.c_void_p * L)(*[t.data_ptr() for t in levels])
    ns = (ctypes.c_uint64 * L)(*level_n)
    args = [ctypes.cast(ptrs, ctypes.c_void_p), ctypes.cast(ns, ctypes.c_void_p), L, rids.data_ptr(),
            keys.data_ptr(), keys.numel(), out.data_ptr(), _stream_ptr(stream)]
    if direct:
        _check(_lib.dpg_btree_lookup_direct(*args), "dpg_btree_lookup_direct")
    else:
        _check(_lib.dpg_btree_lookup(*args, log2_run), "dpg_btree_lookup")
    return out


def dpg_get_unique_id() -> bytes:
    """An NCCL unique id for dpg_comm_create (make on one rank, send to all)."""
    b = (ctypes.c_uint8 * 128)()
    _check(_lib.dpg_get_unique_id(b), "dpg_get_unique_id")
    return bytes(b)


def dpg_comm_create(uid: bytes, nranks: int, rank: int) -> int:
    """The library's own communicator on the current device (collective)."""
    c = ctypes.c_void_p()
    u = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(_lib.dpg_comm_create(u, nranks, rank, ctypes.byref(c)), "dpg_comm_create")
    return int(c.value)


def dpg_comm_destroy(comm: int) -> None:
    _check(_lib.dpg_comm_destroy(ctypes.c_void_p(comm)), "dpg_comm_destroy")


def dpg_retrieve_dist(comm: int, src_shard, n_src_total: int, rids, dst=None, stream=None):
    """The multi-GPU retrieval behind the C ABI (collective over comm): rows
    src_global[rids] for this rank's block; src_shard = this rank's records."""
    torch = _torch()
    src_shard = _records(src_shard, "src_shard")
    rec = src_shard.shape[1]
    if rids.dtype != torch.int64 or not rids.is_cuda or not rids.is_contiguous():
        raise TypeError("rids must be a contiguous CUDA int64 tensor")
    if dst is None:
        dst = torch.empty((rids.numel(), rec), dtype=torch.uint8, device=rids.device)
    _check(_lib.dpg_retrieve_dist(ctypes.c_void_p(comm), src_shard.data_ptr(), rec, n_src_total,
                                  rids.data_ptr(), rids.numel(), dst.data_ptr(),
                                  _stream_ptr(stream)), "dpg_retrieve_dist")
    return dst


def dpg_retrieve_dist_loopback(src_shards, n_src_total: int, rids_list, dsts=None, stream=None):
    """The multi-GPU exchange for P = len(src_shards) virtual ranks on this GPU
    (dpg_retrieve_dist_loopback): rank r owns src_shards[r] (uint8 [S_r, rec]),
    asks for rids_list[r] (int64/uint64 CUDA) and receives dsts[r]."""
    torch = _torch()
    P = len(src_shards)
    if len(rids_list) != P:
        raise ValueError("one rid list per rank")
    shards = [_records(t, "src_shard") for t in src_shards]
    rec = shards[0].shape[1]
    rl = []
    for r in rids_list:
        if r.dtype not in (torch.int64, torch.uint64) or not r.is_contiguous():
            raise TypeError("rids must be contiguous CUDA int64/uint64")
        rl.append(r)
    if dsts is None:
        dsts = [torch.empty((r.numel(), rec), dtype=torch.uint8, device=r.device) for r in rl]
    arr_p = (ctypes.c_void_p * P)
    arr_u = (ctypes.c_uint64 * P)
    _check(_lib.dpg_retrieve_dist_loopback(
        P, arr_p(*[t.data_ptr() for t in shards]), rec, n_src_total,
        arr_p(*[r.data_ptr() for r in rl]), arr_u(*[r.numel() for r in rl]),
        arr_p(*[d.data_ptr() for d in dsts]), _stream_ptr(stream)), "dpg_retrieve_dist_loopback")
    return dsts


def ipc_alloc(nbytes: int) -> tuple[int, bytes]:
    """A device buffer (library-owned) and its 64-byte IPC handle."""
    p = ctypes.c_void_p()
    h = (ctypes.c_uint8 * 64)()
    _check(_lib.dpg_ipc_alloc(nbytes, ctypes.byref(p), h), "dpg_ipc_alloc")
    return int(p.value), bytes(h)


def ipc_open(handle: bytes) -> int:
    """A peer process's buffer mapped into this one (device address)."""
    p = ctypes.c_void_p()
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    _check(_lib.dpg_ipc_open(h, ctypes.byref(p)), "dpg_ipc_open")
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(_lib.dpg_ipc_close(ctypes.c_void_p(ptr)), "dpg_ipc_close")


def ipc_free(ptr: int) -> None:
    _check(_lib.dpg_ipc_free(ctypes.c_void_p(ptr)), "dpg_ipc_free")


def dpg_fk_join_sort(fact, fk_col, dim, out=None, stream=None):
    """DPG-Sort join: rows fact[rid_R] ++ dim[fk] in stable fk order."""
    torch = _torch()
    fact = _records(fact, "fact")
    dim = _records(dim, "dim")
    fk_col = _rid_tensor(fk_col, "fk_col")
    n_fact, fact_bytes = fact.shape
    n_dim, rec = dim.shape
    if fk_col.numel() != n_fact:
        raise ValueError("fk_col must have one entry per fact row")
    if out is None:
        out = torch.empty((n_fact, fact_bytes + rec), dtype=torch.uint8, device=dim.device)
    _check(_lib.dpg_fk_join_sort(fact.data_ptr(), fact_bytes, n_fact, fk_col.data_ptr(),
                                 dim.data_ptr(), rec, n_dim, out.data_ptr(), _stream_ptr(stream)),
           "dpg_fk_join_sort")
    return out


def dpg_sort_rids(src, key_off: int, key_bytes: int, rids=None, stream=None):
    """Phases 1-2 of three-phase sorting: the rids of src's
    records in stable order of their key (key_bytes bytes at key_off)."""
    torch = _torch()
    src = _records(src, "src")
    n, rec = src.shape
    if rids is None:
        rids = torch.empty(n, dtype=torch.int32, device=src.device)
    _check(_lib.dpg_sort_rids(src.data_ptr(), rec, n, key_off, key_bytes, rids.data_ptr(),
                              _stream_ptr(stream)), "dpg_sort_rids")
    return rids


def dpg_sort(src, key_off: int, key_bytes: int, dst=None, stream=None):
    """The DPG sort: src's records sorted by key, with
    DPG record retrieval as the record-copy phase."""
    torch = _torch()
    src = _records(src, "src")
    n, rec = src.shape
    if dst is None:
        dst = torch.empty((n, rec), dtype=torch.uint8, device=src.device)
    _check(_lib.dpg_sort(src.data_ptr(), rec, n, key_off, key_bytes, dst.data_ptr(),
                         _stream_ptr(stream)), "dpg_sort")
    return dst


def dpg_release_cache():
    _lib.dpg_release_cache()


def dpg_sync_status(stream=None):
    """Synchronise the stream; raise DPGError(DPG_ERR_RID_RANGE, index) if a
    rid was out of range since the last check."""
    idx = ctypes.c_uint64(0)
    s = _lib.dpg_sync_status(_stream_ptr(stream), ctypes.byref(idx))
    if s == DPG_ERR_RID_RANGE:
        raise DPGError(s, "dpg_sync_status", int(idx.value))
    _check(s, "dpg_sync_status")


def raw_lib():
    """The loaded ctypes library (tests of the C ABI itself)."""
    return _lib
