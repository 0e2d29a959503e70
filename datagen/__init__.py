"""Seeded synthetic inputs for DPG record retrieval (shared by both sides).

Holds none of the method's arithmetic: only record bytes, rid sequences and
foreign keys, produced by the counter-based generators of ``datagen/gen.c``
(reading A12 in DESIGN.md).  Seeds are 0 everywhere (reading A13); every
array has its own stream id, listed in :data:`STREAMS` and echoed in the
bench JSON.

Workloads (BASELINE.json ``configs``):

* ``c1``  65,536 x 100 B, rids = uniform random permutation (uint32)
* ``c2``  1,048,576 x 100 B Datamation-shaped records (10-byte key at offset 0
  ++ 90-byte payload, all random bytes); rids = stable argsort of the keys
  (ties by ascending rid, reading A10) -- the sort's phase 3
* ``c3a`` 16,777,216 x rec, rec in {8,16,32,64,128,256}, rids = permutation
* ``c3b`` same, rids iid uniform with replacement
* ``c2L`` 16,777,216 x 100 B, rids = permutation (SURVEY 8(d)'s "2L" row)
* ``c4``  dimension 16,777,216 x 64 B; fact 67,108,864 x (uint32 fk uniform in
  [0, 2^24) ++ 16-byte payload) -- the DPG-Move join
* ``c4x`` config 4 with the paper's non-uniform foreign keys:
  fk = min(n_dim - 1, floor(n_dim * exp(c * (r >> 10)))), r a uniform 31-bit
  draw (the range of UNIX random()), c = -1e-7 (reading A18 in DESIGN.md)
* ``c5``  2^30 x 100 B, rids = Feistel permutation (uint64), evaluated pointwise

These synthetic inputs stand in for the paper's workloads (Datamation
benchmark records, the record-size sweep, uniform foreign keys); no benchmark
item or dataset is reproduced.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libdpggen.so")
_lib = None

SEED = 0
# stream ids: (config, array) -> sid
STREAMS = {
    ("c1", "src"): 0x101, ("c1", "rids"): 0x102,
    ("c2", "src"): 0x201,
    ("c3", "src"): 0x301, ("c3a", "rids"): 0x302, ("c3b", "rids"): 0x303,
    ("c4", "dim"): 0x401, ("c4", "fact"): 0x402, ("c4", "fk"): 0x403, ("c4x", "fk"): 0x404,
    ("c5", "src"): 0x501, ("c5", "rids"): 0x502,
    ("test", "src"): 0x901, ("test", "rids"): 0x902,
    ("h1", "keys"): 0x601, ("h1", "queries"): 0x602, ("h1", "absent"): 0x603,
}

C3_RECS = (8, 16, 32, 64, 128, 256)


_CU_SRC = os.path.join(_HERE, "gen_cuda.cu")
_CU_LIB = os.path.join(_HERE, "libdpggen_cuda.so")
_culib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-std=c11", "-fopenmp", "-shared", "-fPIC",
                               _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    if force or not os.path.exists(_CU_LIB) or os.path.getmtime(_CU_LIB) < os.path.getmtime(_CU_SRC):
        tmp = _CU_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-shared",
                               "-Xcompiler", "-fPIC", "-cudart", "static",
                               "-gencode", "arch=compute_100a,code=sm_100a", _CU_SRC, "-o", tmp])
        os.replace(tmp, _CU_LIB)
    return _LIB


def _load_cuda():
    global _culib
    if _culib is None:
        build()
        lib = ctypes.CDLL(_CU_LIB)
        U, P = ctypes.c_uint64, ctypes.c_void_p
        lib.gen_bytes_cuda.argtypes = [U, U, U, U, P, P]
        lib.gen_feistel_cuda.argtypes = [U, U, ctypes.c_uint, ctypes.c_uint, U, U, U, P, P]
        _culib = lib
    return _culib


def random_bytes_cuda(t, sid: int, seed: int = SEED, offset: int = 0):
    """Fill the CUDA uint8 tensor t with bytes [offset, offset + t.numel()) of
    stream sid (same values as random_bytes; offset and size multiples of 8)."""
    import torch
    s = torch.cuda.current_stream().cuda_stream
    if _load_cuda().gen_bytes_cuda(seed, sid, offset, t.numel(), t.data_ptr(), s):
        raise RuntimeError("gen_bytes_cuda failed")
    return t


def feistel_cuda(n: int, first: int, count: int, sid: int, seed: int = SEED, rounds: int = 6):
    """Elements [first, first+count) of the Feistel permutation of [0, n) as a
    CUDA int64 tensor (same values as feistel)."""
    import torch
    bits = max(2, (n - 1).bit_length())
    bits += bits & 1
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    if _load_cuda().gen_feistel_cuda(seed, sid, bits, rounds, n, first, count, out.data_ptr(), s):
        raise RuntimeError("gen_feistel_cuda failed")
    return out


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        U, P = ctypes.c_uint64, ctypes.c_void_p
        lib.gen_word.argtypes = [U, U, U]
        lib.gen_word.restype = U
        lib.gen_bytes.argtypes = [U, U, U, U, P]
        lib.gen_permutation_u32.argtypes = [U, U, U, P]
        lib.gen_uniform_u32.argtypes = [U, U, U, U, P]
        lib.gen_feistel_u64.argtypes = [U, U, ctypes.c_uint, ctypes.c_uint, U, U, U, P]
        lib.gen_hash_index.argtypes = [P, U, ctypes.c_uint, P, P]
        lib.gen_hash_index.restype = U
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def word(sid: int, k: int, seed: int = SEED) -> int:
    return int(_load().gen_word(seed, sid, k))


def random_bytes(n: int, sid: int, seed: int = SEED, offset: int = 0, out=None) -> np.ndarray:
    out = np.empty(n, dtype=np.uint8) if out is None else out
    assert out.dtype == np.uint8 and out.flags.c_contiguous and out.size == n
    _load().gen_bytes(seed, sid, offset, n, _p(out))
    return out


def records(n: int, rec: int, sid: int, seed: int = SEED, out=None) -> np.ndarray:
    """n records of rec uniformly random bytes: uint8 [n, rec]."""
    flat = random_bytes(n * rec, sid, seed, out=None if out is None else out.reshape(-1))
    return flat.reshape(n, rec)


def permutation(n: int, sid: int, seed: int = SEED) -> np.ndarray:
    """Uniformly random permutation of [0, n) as uint32 (Fisher-Yates)."""
    assert n < 2 ** 32
    out = np.empty(n, dtype=np.uint32)
    _load().gen_permutation_u32(seed, sid, n, _p(out))
    return out


def uniform(n: int, bound: int, sid: int, seed: int = SEED) -> np.ndarray:
    """n iid uniform draws in [0, bound) as uint32 (with replacement)."""
    assert 0 < bound <= 2 ** 32
    out = np.empty(n, dtype=np.uint32)
    _load().gen_uniform_u32(seed, sid, n, bound, _p(out))
    return out


def feistel(n: int, first: int, count: int, sid: int, seed: int = SEED,
            rounds: int = 6) -> np.ndarray:
    """Elements [first, first+count) of a keyed Feistel permutation of [0, n), uint64."""
    bits = max(2, (n - 1).bit_length())
    bits += bits & 1
    out = np.empty(count, dtype=np.uint64)
    _load().gen_feistel_u64(seed, sid, bits, rounds, n, first, count, _p(out))
    return out


def exp_fk(n: int, n_dim: int, sid: int, seed: int = SEED, c: float = -1e-7) -> np.ndarray:
    """The paper's exponential join keys, exp(c * (random() >> 10))
    with random() a uniform 31-bit draw, scaled to the key domain [0, n_dim)
    (reading A18): uint32, concentrated in the top ~19% of the domain with
    density proportional to 1/key."""
    r = uniform(n, 2 ** 31, sid, seed).astype(np.int64)
    y = np.exp(c * (r >> 10).astype(np.float64))
    return np.minimum(n_dim - 1, np.floor(n_dim * y)).astype(np.uint32)


def hash_index(keys: np.ndarray, m_log2: int):
    """The hash index of the batch lookup over (keys[j], rid j) (gen.c
    gen_hash_index): (table uint32 [2^m_log2, 4], pool uint32 [P, 4])."""
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    table = np.empty((1 << m_log2, 4), dtype=np.uint32)
    pool = np.empty((max(1, keys.size), 4), dtype=np.uint32)
    n_pool = _load().gen_hash_index(_p(keys), keys.size, m_log2, _p(table), _p(pool))
    return table, pool[:max(1, n_pool)].copy()


def hash_workload(n_keys: int, m_log2: int, n_queries: int, absent_per_mille: int = 50):
    """Batch lookup workload: distinct uint32 keys (a 32-bit
    Feistel permutation), their index, and queries drawn uniformly from the
    keys with ~absent_per_mille / 1000 of them replaced by absent keys."""
    keys = feistel(1 << 32, 0, n_keys, STREAMS[("h1", "keys")]).astype(np.uint32)
    table, pool = hash_index(keys, m_log2)
    q = keys[uniform(n_queries, n_keys, STREAMS[("h1", "queries")]).astype(np.int64)]
    n_abs = n_queries * absent_per_mille // 1000
    if n_abs:
        pos = uniform(n_abs, n_queries, STREAMS[("h1", "absent")]).astype(np.int64)
        q[pos] = feistel(1 << 32, n_keys, n_abs, STREAMS[("h1", "keys")]).astype(np.uint32)
    return {"keys": keys, "table": table, "pool": pool, "queries": q}


BTREE_FANOUT = 16


def btree_index(keys: np.ndarray):
    """The enhanced B+-tree of the batch lookup (every slot used)
    over (keys[j], rid j): level 0 = the keys sorted (with their rids), level
    t = every 16th entry of level t-1 (the first key of each node below),
    up to a top level of <= 16 entries.  Returns (levels, rids): levels[0] is
    the sorted keys (uint32), rids[j] the rid of levels[0][j]."""
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    order = np.argsort(keys, kind="stable")
    levels = [keys[order]]
    while levels[-1].size > BTREE_FANOUT:
        levels.append(np.ascontiguousarray(levels[-1][::BTREE_FANOUT]))
    return levels, order.astype(np.uint32)


def stable_key_argsort(recs: np.ndarray, key_len: int = 10) -> np.ndarray:
    """Stable argsort of the records' key bytes (offset 0, unsigned
    lexicographic), ties by ascending rid (reading A10).  Part of the input
    generator for config 2: the sort's phases 1-2 are not the
    retrieval path; only their result (the rid sequence) is an input."""
    assert key_len <= 10
    keys = np.zeros((recs.shape[0], 10), dtype=np.uint8)
    keys[:, :key_len] = recs[:, :key_len]
    hi = keys[:, :8].copy().view(">u8").reshape(-1)
    lo = keys[:, 8:10].copy().view(">u2").reshape(-1)
    return np.lexsort((lo, hi)).astype(np.uint32)


def make(config: str, rec: int | None = None, scale: int = 1) -> dict:
    """Build a named workload.  ``scale`` > 1 divides the sizes (tests)."""
    if config == "c1":
        n = 65536 // scale
        return {"src": records(n, 100, STREAMS[("c1", "src")]),
                "rids": permutation(n, STREAMS[("c1", "rids")])}
    if config == "c2":
        n = 1048576 // scale
        src = records(n, 100, STREAMS[("c2", "src")])
        return {"src": src, "rids": stable_key_argsort(src, 10)}
    if config in ("c3a", "c3b"):
        assert rec in C3_RECS
        n = 16777216 // scale
        src = records(n, rec, STREAMS[("c3", "src")])
        if config == "c3a":
            rids = permutation(n, STREAMS[("c3a", "rids")])
        else:
            rids = uniform(n, n, STREAMS[("c3b", "rids")])
        return {"src": src, "rids": rids}
    if config == "c2L":
        # SURVEY 8(d) row "2L": config 2's record size on config 3's scale,
        # 16,777,216 x 100 B, rids = a uniform random permutation
        n = 16777216 // scale
        return {"src": records(n, 100, STREAMS[("c3", "src")]),
                "rids": permutation(n, STREAMS[("c3a", "rids")])}
    if config in ("c4", "c4x"):
        n_dim = 16777216 // scale
        n_fact = 67108864 // scale
        fk = uniform(n_fact, n_dim, STREAMS[("c4", "fk")]) if config == "c4" else \
            exp_fk(n_fact, n_dim, STREAMS[("c4x", "fk")])
        return {"dim": records(n_dim, 64, STREAMS[("c4", "dim")]),
                "fact": records(n_fact, 16, STREAMS[("c4", "fact")]), "fk": fk}
    raise KeyError(config)
