"""ctypes loader for the plain-C RecSplit oracle (``oracle/recsplit_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs, never by the product
package ``paper_2212_09562_b200``.  Shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "recsplit_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, E_INVALID, E_DUPLICATE, E_NOMEM, E_FORMAT, E_SEED_CAP = 0, -1, -2, -3, -5, -6


def compile_oracle(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no intrinsics, no -march)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC,
                               "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(compile_oracle())
        u64, u32, i32, dbl = C.c_uint64, C.c_uint32, C.c_int, C.c_double
        P64, P8 = C.POINTER(C.c_uint64), C.POINTER(C.c_uint8)
        L.oracle_remix.restype, L.oracle_remix.argtypes = u64, [u64]
        L.oracle_mhc.restype, L.oracle_mhc.argtypes = None, [u64, u64, P64, P64]
        L.oracle_remap.restype, L.oracle_remap.argtypes = u32, [u64, u64]
        L.oracle_shape.restype = None
        L.oracle_shape.argtypes = [u32] + [C.POINTER(C.c_uint32)] * 4
        L.oracle_parts.restype, L.oracle_parts.argtypes = i32, [u32, u32, C.POINTER(C.c_uint32)]
        L.oracle_find_split.restype, L.oracle_find_split.argtypes = i32, [u32, P64, u32, P64]
        L.oracle_leaf_bf.restype, L.oracle_leaf_bf.argtypes = i32, [P64, u32, P64]
        L.oracle_leaf_rf.restype, L.oracle_leaf_rf.argtypes = i32, [P64, P8, u32, P64]
        L.oracle_rot.restype, L.oracle_rot.argtypes = u64, [u32, u32, u64]
        L.oracle_split_prob.restype, L.oracle_split_prob.argtypes = dbl, [u32, u32]
        L.oracle_bij_prob_bf.restype, L.oracle_bij_prob_bf.argtypes = dbl, [u32]
        L.oracle_bij_prob_rf.restype, L.oracle_bij_prob_rf.argtypes = dbl, [u32]
        L.oracle_necklaces.restype, L.oracle_necklaces.argtypes = dbl, [u32]
        L.oracle_golomb_tau.restype, L.oracle_golomb_tau.argtypes = i32, [dbl]
        L.oracle_tau.restype, L.oracle_tau.argtypes = i32, [u32, u32, i32]
        L.oracle_build_ex.restype = i32
        L.oracle_build_ex.argtypes = [P64, u64, u32, u32, i32, u64, i32, C.POINTER(P8),
                                      C.POINTER(u64), C.POINTER(P64), C.POINTER(u64)]
        L.oracle_bucket_values.restype = i32
        L.oracle_bucket_values.argtypes = [P64, u64, u32, i32, u64, P64, C.POINTER(u64)]
        L.oracle_query_many.restype = i32
        L.oracle_query_many.argtypes = [P8, u64, P64, u64, P64]
        L.oracle_free.restype, L.oracle_free.argtypes = None, [C.c_void_p]
        L.oracle_mhc_string.restype = None
        L.oracle_murmur3_x64_128.restype = None
        L.oracle_murmur3_x64_128.argtypes = [P8, u64, u32, P64, P64]
        L.oracle_mhc_string.argtypes = [P8, u64, u64, P64, P64]
        L.oracle_build_strings.restype = i32
        L.oracle_build_strings.argtypes = [P8, P64, u64, u32, u32, i32, u64, i32, C.POINTER(P8), C.POINTER(u64)]
        L.oracle_query_strings.restype = i32
        L.oracle_query_strings.argtypes = [P8, u64, P8, P64, u64, P64]
        _lib = L
    return _lib


def _p64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def remix(z: int) -> int:
    return lib().oracle_remix(z)


def mhc(key: int, g: int = 0) -> tuple[int, int]:
    hi, lo = C.c_uint64(), C.c_uint64()
    lib().oracle_mhc(key, g, C.byref(hi), C.byref(lo))
    return hi.value, lo.value


def remap(h: int, r: int) -> int:
    return lib().oracle_remap(h, r)


def rot(m: int, r: int, x: int) -> int:
    return lib().oracle_rot(m, r, x)


def shape(leaf: int) -> tuple[int, int, int, int]:
    v = [C.c_uint32() for _ in range(4)]
    lib().oracle_shape(leaf, *[C.byref(x) for x in v])
    return tuple(x.value for x in v)


def parts(leaf: int, s: int) -> list[int]:
    buf = (C.c_uint32 * 64)()
    f = lib().oracle_parts(leaf, s, buf)
    return list(buf[:f])


def split_prob(leaf: int, s: int) -> float:
    return lib().oracle_split_prob(leaf, s)


def bij_prob(m: int, rf: bool) -> float:
    return lib().oracle_bij_prob_rf(m) if rf else lib().oracle_bij_prob_bf(m)


def necklaces(m: int) -> float:
    return lib().oracle_necklaces(m)


def golomb_tau(p: float) -> int:
    return lib().oracle_golomb_tau(p)


def tau(leaf: int, s: int, rf: bool) -> int:
    return lib().oracle_tau(leaf, s, int(rf))


def find_split(leaf: int, lo) -> int:
    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    out = C.c_uint64()
    rc = lib().oracle_find_split(leaf, _p64(lo), len(lo), C.byref(out))
    if rc:
        raise RuntimeError(f"oracle_find_split rc={rc}")
    return out.value


def leaf_bf(lo) -> int:
    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    out = C.c_uint64()
    rc = lib().oracle_leaf_bf(_p64(lo), len(lo), C.byref(out))
    if rc:
        raise RuntimeError(f"oracle_leaf_bf rc={rc}")
    return out.value


def leaf_rf(lo, isb) -> int:
    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    isb = np.ascontiguousarray(isb, dtype=np.uint8)
    out = C.c_uint64()
    rc = lib().oracle_leaf_rf(_p64(lo), isb.ctypes.data_as(C.POINTER(C.c_uint8)), len(lo),
                              C.byref(out))
    if rc:
        raise RuntimeError(f"oracle_leaf_rf rc={rc}")
    return out.value


class OracleError(RuntimeError):
    def __init__(self, rc: int, what: str):
        super().__init__(f"{what} failed rc={rc}")
        self.rc = rc


def build(keys, leaf: int, bucket: int, rf: bool = True, g: int = 0, threads: int = 1,
          values: bool = False):
    """Serialized MPHF bytes (and optionally the node values in bucket/preorder)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    out = C.POINTER(C.c_uint8)()
    size = C.c_uint64()
    vals = C.POINTER(C.c_uint64)()
    nv = C.c_uint64()
    rc = lib().oracle_build_ex(_p64(keys), len(keys), leaf, bucket, int(rf), g, threads,
                               C.byref(out), C.byref(size),
                               C.byref(vals) if values else None, C.byref(nv) if values else None)
    if rc:
        raise OracleError(rc, "oracle_build")
    blob = C.string_at(out, size.value)
    lib().oracle_free(out)
    if not values:
        return blob
    v = np.ctypeslib.as_array(vals, shape=(nv.value,)).copy() if nv.value else np.zeros(0, np.uint64)
    lib().oracle_free(vals)
    return blob, v


def bucket_values(keys, leaf: int, rf: bool = True, g: int = 0) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    buf = np.zeros(max(1, 4 * len(keys) + 4), dtype=np.uint64)
    nv = C.c_uint64()
    rc = lib().oracle_bucket_values(_p64(keys), len(keys), leaf, int(rf), g, _p64(buf), C.byref(nv))
    if rc:
        raise OracleError(rc, "oracle_bucket_values")
    return buf[: nv.value].copy()


def query_many(blob: bytes, keys) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.zeros(len(keys), dtype=np.uint64)
    b = np.frombuffer(blob, dtype=np.uint8)
    rc = lib().oracle_query_many(b.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob), _p64(keys),
                                 len(keys), _p64(out))
    if rc:
        raise OracleError(rc, "oracle_query_many")
    return out


# ---------------------------------------------------------------- string keys (N4) --

def _p8(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def murmur3_x64_128(s: bytes, seed: int = 0) -> tuple[int, int]:
    buf = np.frombuffer(s, dtype=np.uint8) if len(s) else np.zeros(1, np.uint8)
    h1, h2 = C.c_uint64(), C.c_uint64()
    lib().oracle_murmur3_x64_128(_p8(buf), len(s), seed, C.byref(h1), C.byref(h2))
    return h1.value, h2.value


def mhc_string(s: bytes, g: int = 0) -> tuple[int, int]:
    buf = np.frombuffer(s, dtype=np.uint8) if len(s) else np.zeros(1, np.uint8)
    hi, lo = C.c_uint64(), C.c_uint64()
    lib().oracle_mhc_string(_p8(buf), len(s), g, C.byref(hi), C.byref(lo))
    return hi.value, lo.value


def build_strings(data, offsets, leaf: int, bucket: int, rf: bool = True, g: int = 0, threads: int = 1) -> bytes:
    data = np.ascontiguousarray(data, dtype=np.uint8)
    if data.size == 0:
        data = np.zeros(1, np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    out = C.POINTER(C.c_uint8)()
    size = C.c_uint64()
    rc = lib().oracle_build_strings(_p8(data), _p64(offsets), len(offsets) - 1, leaf, bucket, int(rf), g, threads,
                                    C.byref(out), C.byref(size))
    if rc:
        raise OracleError(rc, "oracle_build_strings")
    blob = C.string_at(out, size.value)
    lib().oracle_free(out)
    return blob


def query_strings(blob: bytes, data, offsets) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.uint8)
    if data.size == 0:
        data = np.zeros(1, np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = len(offsets) - 1
    out = np.zeros(n, dtype=np.uint64)
    b = np.frombuffer(blob, dtype=np.uint8)
    rc = lib().oracle_query_strings(_p8(b), len(blob), _p8(data), _p64(offsets), n, _p64(out))
    if rc:
        raise OracleError(rc, "oracle_query_strings")
    return out
