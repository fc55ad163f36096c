"""Thin Python binding of the B200-native RecSplit builder (``include/recsplit.h``).

Argument marshalling only: every construction step runs in the CUDA kernels of
``lib/librecsplit_b200.so``.  There is no CPU fallback -- if the library is
missing or no CUDA device is usable, calls raise ``RecSplitError``.
PyTorch is used only to pass device memory and streams (``build_device``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RECSPLIT_LIB", os.path.join(_HERE, "lib", "librecsplit_b200.so"))

OK, E_INVALID, E_DUPLICATE, E_NOMEM, E_CUDA, E_FORMAT, E_SEED_CAP = 0, -1, -2, -3, -4, -5, -6

# Every symbol include/recsplit.h declares.
SYMBOLS = [
    "recsplit_version", "recsplit_max_bucket_keys", "recsplit_build", "recsplit_build_ex",
    "recsplit_build_device", "recsplit_build_values", "recsplit_query", "recsplit_query_many",
    "recsplit_bits_per_key", "recsplit_search_leaves", "recsplit_search_splits", "recsplit_tau",
    "recsplit_free", "recsplit_free_ptr", "recsplit_last_error", "recsplit_shard_begin",
    "recsplit_shard_min_step", "recsplit_shard_finish", "recsplit_stitch", "recsplit_shard_free",
    "recsplit_shard_globals", "recsplit_query_device", "recsplit_build_strings", "recsplit_query_strings",
    "recsplit_open", "recsplit_handle_query_many", "recsplit_handle_query_device", "recsplit_close",
    "recsplit_check_bijective_device", "recsplit_route_keys", "recsplit_bucket_histogram",
    "recsplit_balanced_cuts", "recsplit_trim",
]


class RecSplitError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"recsplit error {code}: {msg}")
        self.code = code


class Bytes(C.Structure):
    _fields_ = [("data", C.POINTER(C.c_uint8)), ("size", C.c_size_t)]


class Options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("rotation_fitting", C.c_uint32),
                ("global_seed", C.c_uint64), ("device", C.c_int32), ("virtual_shards", C.c_uint32),
                ("reserved", C.c_uint32), ("total_keys", C.c_uint64),
                ("bucket_cuts", C.POINTER(C.c_uint64))]


class Stats(C.Structure):
    _fields_ = [("t_total", C.c_double), ("t_h2d", C.c_double), ("t_partition", C.c_double),
                ("t_tree", C.c_double), ("t_search", C.c_double * 4), ("t_reorder", C.c_double),
                ("t_encode", C.c_double), ("t_d2h", C.c_double), ("algo_evals", C.c_uint64 * 4),
                ("nodes", C.c_uint64 * 4), ("data_bits", C.c_uint64), ("index_bits", C.c_uint64),
                ("kernel_launches", C.c_uint32), ("max_bucket", C.c_uint32), ("exec_evals", C.c_uint64 * 4),
                ("t_search_tree", C.c_double), ("t_device", C.c_double), ("graph_replay", C.c_uint32),
                ("reserved0", C.c_uint32)]

    def as_dict(self) -> dict:
        return {
            "t_total": self.t_total, "t_h2d": self.t_h2d, "t_partition": self.t_partition,
            "t_tree": self.t_tree, "t_search": list(self.t_search), "t_reorder": self.t_reorder,
            "t_encode": self.t_encode, "t_d2h": self.t_d2h, "algo_evals": list(self.algo_evals),
            "nodes": list(self.nodes), "data_bits": self.data_bits, "index_bits": self.index_bits,
            "kernel_launches": self.kernel_launches, "max_bucket": self.max_bucket,
            "exec_evals": list(self.exec_evals), "t_search_tree": self.t_search_tree,
            "t_device": self.t_device, "graph_replay": self.graph_replay,
        }


_lib = None


def lib():
    """Load the CUDA library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RecSplitError(E_CUDA, f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P64, P8, P32 = C.POINTER(C.c_uint64), C.POINTER(C.c_uint8), C.POINTER(C.c_uint32)
        u32, u64, sz, i32 = C.c_uint32, C.c_uint64, C.c_size_t, C.c_int
        L.recsplit_version.restype = i32
        L.recsplit_max_bucket_keys.restype = u32
        L.recsplit_build.argtypes = [P64, sz, u32, u32, C.POINTER(Bytes)]
        L.recsplit_build_ex.argtypes = [P64, sz, u32, u32, C.POINTER(Options), C.POINTER(Bytes),
                                        C.POINTER(Stats)]
        L.recsplit_build_device.argtypes = [C.c_void_p, sz, u32, u32, C.POINTER(Options), C.c_void_p,
                                            C.POINTER(Bytes), C.POINTER(Stats)]
        L.recsplit_build_values.argtypes = [P64, sz, u32, u32, C.POINTER(Options), C.POINTER(Bytes),
                                            C.POINTER(P64), C.POINTER(sz)]
        L.recsplit_query.argtypes = [P8, sz, u64, P64]
        L.recsplit_query_many.argtypes = [P8, sz, P64, sz, P64]
        L.recsplit_bits_per_key.argtypes = [P8, sz, C.POINTER(C.c_double)]
        L.recsplit_query_device.argtypes = [P8, sz, C.c_void_p, sz, C.c_void_p, C.c_void_p]
        L.recsplit_query_device.restype = i32
        L.recsplit_build_strings.argtypes = [P8, P64, sz, u32, u32, C.POINTER(Options), C.POINTER(Bytes),
                                             C.POINTER(Stats)]
        L.recsplit_build_strings.restype = i32
        L.recsplit_query_strings.argtypes = [P8, sz, P8, P64, sz, P64]
        L.recsplit_query_strings.restype = i32
        L.recsplit_search_leaves.argtypes = [P64, P8, P32, u32, u32, P64]
        L.recsplit_search_splits.argtypes = [P64, P32, u32, u32, P64]
        L.recsplit_tau.argtypes = [u32, u32, u32]
        L.recsplit_free.argtypes = [C.POINTER(Bytes)]
        L.recsplit_free.restype = None
        L.recsplit_free_ptr.argtypes = [C.c_void_p]
        L.recsplit_free_ptr.restype = None
        L.recsplit_last_error.restype = C.c_char_p
        L.recsplit_shard_begin.argtypes = [C.c_void_p, sz, u32, u32, C.POINTER(Options), C.c_int32, C.c_int32,
                                           C.c_void_p, C.POINTER(C.c_void_p), P64]
        L.recsplit_shard_min_step.argtypes = [C.c_void_p, P64, C.POINTER(C.c_int64)]
        L.recsplit_shard_finish.argtypes = [C.c_void_p, C.c_int64, C.POINTER(Bytes)]
        L.recsplit_stitch.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int32, C.POINTER(Bytes)]
        L.recsplit_shard_free.argtypes = [C.c_void_p]
        L.recsplit_shard_free.restype = None
        L.recsplit_shard_globals.argtypes = [P64, C.c_int32, C.c_int32, P64]
        L.recsplit_open.argtypes = [P8, sz, C.c_int32, C.POINTER(C.c_void_p)]
        L.recsplit_open.restype = i32
        L.recsplit_handle_query_many.argtypes = [C.c_void_p, P64, sz, P64]
        L.recsplit_handle_query_many.restype = i32
        L.recsplit_handle_query_device.argtypes = [C.c_void_p, C.c_void_p, sz, C.c_void_p, C.c_void_p]
        L.recsplit_handle_query_device.restype = i32
        L.recsplit_check_bijective_device.argtypes = [C.c_void_p, sz, P64, C.c_void_p]
        L.recsplit_check_bijective_device.restype = i32
        L.recsplit_route_keys.argtypes = [C.c_void_p, sz, u64, u32, C.POINTER(Options), C.c_int32, C.c_void_p,
                                          C.c_void_p, P64]
        L.recsplit_route_keys.restype = i32
        L.recsplit_bucket_histogram.argtypes = [C.c_void_p, sz, u64, u32, C.POINTER(Options), C.c_void_p, C.c_void_p]
        L.recsplit_bucket_histogram.restype = i32
        L.recsplit_balanced_cuts.argtypes = [P32, u64, u32, u32, C.c_int32, P64]
        L.recsplit_balanced_cuts.restype = i32
        L.recsplit_close.argtypes = [C.c_void_p]
        L.recsplit_close.restype = None
        L.recsplit_trim.argtypes = []
        L.recsplit_trim.restype = i32
        for name in ("recsplit_shard_begin", "recsplit_shard_min_step", "recsplit_shard_finish", "recsplit_stitch",
                     "recsplit_shard_globals"):
            getattr(L, name).restype = i32
        for name in ("recsplit_build", "recsplit_build_ex", "recsplit_build_device", "recsplit_build_values",
                     "recsplit_query", "recsplit_query_many", "recsplit_bits_per_key",
                     "recsplit_search_leaves", "recsplit_search_splits", "recsplit_tau"):
            getattr(L, name).restype = i32
        _lib = L
    return _lib


def _check(rc: int):
    if rc < 0:
        raise RecSplitError(rc, lib().recsplit_last_error().decode())
    return rc


def _p64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _opts(rotation_fitting: bool, global_seed: int, device: int, virtual_shards: int, total_keys: int = 0,
          cuts=None):
    """Options struct; `cuts` (uint64 array of world + 1 bucket indices) must outlive the call."""
    return Options(C.sizeof(Options), int(bool(rotation_fitting)), global_seed, device, virtual_shards, 0,
                   total_keys, _p64(cuts) if cuts is not None else None)


def _take(b: Bytes) -> bytes:
    out = C.string_at(b.data, b.size)
    lib().recsplit_free(C.byref(b))
    return out


class _Owner:
    """Owns a library result buffer (freed with recsplit_free when collected) and exposes it
    to numpy through the array interface (a read-only view, no copy)."""

    __slots__ = ("holder", "__array_interface__", "__weakref__")

    def __init__(self, b: Bytes):
        self.holder = Bytes(b.data, b.size)
        addr = C.cast(b.data, C.c_void_p).value or 0
        self.__array_interface__ = {"data": (addr, True), "shape": (b.size,), "typestr": "|u1", "version": 3}

    def __del__(self):
        if self.holder.data:
            _lib.recsplit_free(C.byref(self.holder))


def _view(b: Bytes) -> np.ndarray:
    """The library's result buffer as a read-only uint8 array (no copy); released with
    recsplit_free when the array is garbage collected (the array keeps its owner alive)."""
    if not b.size:
        lib().recsplit_free(C.byref(b))
        return np.zeros(0, np.uint8)
    return np.asarray(_Owner(b))


def build(keys, leaf_size: int, bucket_size: int, rotation_fitting: bool = True, global_seed: int = 0,
          device: int = -1, virtual_shards: int = 0, stats: bool = False, cuts=None, copy: bool = True):
    """Build from host keys (uint64 array).  Returns bytes (and a stats dict).  With
    virtual_shards > 1, `cuts` (virtual_shards + 1 bucket indices) sets the shard ranges.
    copy=False: a read-only uint8 numpy view of the library's result buffer instead of bytes."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    b = Bytes()
    st = Stats()
    cuts = None if cuts is None else np.ascontiguousarray(cuts, dtype=np.uint64)
    o = _opts(rotation_fitting, global_seed, device, virtual_shards, cuts=cuts)
    _check(lib().recsplit_build_ex(_p64(keys), len(keys), leaf_size, bucket_size, C.byref(o), C.byref(b),
                                   C.byref(st)))
    blob = _take(b) if copy else _view(b)
    return (blob, st.as_dict()) if stats else blob


def build_device(keys_tensor, leaf_size: int, bucket_size: int, rotation_fitting: bool = True,
                 global_seed: int = 0, stream=None, stats: bool = False, virtual_shards: int = 0,
                 copy: bool = True):
    """Build from a CUDA tensor of keys (int64/uint64 bit patterns) resident in HBM
    (virtual_shards > 1: the bucket-range sharded path on this one device).  copy=False returns
    the serialized MPHF as a read-only uint8 numpy array over the library's buffer (no host
    copy) instead of bytes."""
    import torch

    if not keys_tensor.is_cuda or not keys_tensor.is_contiguous() or keys_tensor.element_size() != 8:
        raise ValueError("keys_tensor must be a contiguous 8-byte CUDA tensor")
    if stream is None:
        stream = torch.cuda.current_stream(keys_tensor.device)
    b = Bytes()
    st = Stats()
    o = _opts(rotation_fitting, global_seed, keys_tensor.device.index, virtual_shards)
    _check(lib().recsplit_build_device(C.c_void_p(keys_tensor.data_ptr()), keys_tensor.numel(), leaf_size,
                                       bucket_size, C.byref(o), C.c_void_p(stream.cuda_stream), C.byref(b),
                                       C.byref(st)))
    blob = _take(b) if copy else _view(b)
    return (blob, st.as_dict()) if stats else blob


def build_values(keys, leaf_size: int, bucket_size: int, rotation_fitting: bool = True,
                 global_seed: int = 0, virtual_shards: int = 0):
    """Diagnostic build: (bytes, node values in bucket order / preorder)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    b = Bytes()
    vp = C.POINTER(C.c_uint64)()
    nv = C.c_size_t()
    o = _opts(rotation_fitting, global_seed, -1, virtual_shards)
    _check(lib().recsplit_build_values(_p64(keys), len(keys), leaf_size, bucket_size, C.byref(o), C.byref(b),
                                       C.byref(vp), C.byref(nv)))
    vals = np.ctypeslib.as_array(vp, shape=(nv.value,)).copy() if nv.value else np.zeros(0, np.uint64)
    lib().recsplit_free_ptr(vp)
    return _take(b), vals


def build_strings(data, offsets, leaf_size: int, bucket_size: int, rotation_fitting: bool = True,
                  global_seed: int = 0, stats: bool = False):
    """Build from string keys: data (uint8) holds key i at data[offsets[i]:offsets[i+1]]."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    if data.size == 0:
        data = np.zeros(1, np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    b = Bytes()
    st = Stats()
    o = _opts(rotation_fitting, global_seed, -1, 0)
    _check(lib().recsplit_build_strings(data.ctypes.data_as(C.POINTER(C.c_uint8)), _p64(offsets), len(offsets) - 1,
                                        leaf_size, bucket_size, C.byref(o), C.byref(b), C.byref(st)))
    blob = _take(b)
    return (blob, st.as_dict()) if stats else blob


def query_strings(blob: bytes, data, offsets) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.uint8)
    if data.size == 0:
        data = np.zeros(1, np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    out = np.zeros(len(offsets) - 1, dtype=np.uint64)
    buf = np.frombuffer(blob, dtype=np.uint8)
    _check(lib().recsplit_query_strings(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob),
                                        data.ctypes.data_as(C.POINTER(C.c_uint8)), _p64(offsets), len(out),
                                        _p64(out)))
    return out


def query(blob: bytes, key: int) -> int:
    out = C.c_uint64()
    buf = np.frombuffer(blob, dtype=np.uint8)
    _check(lib().recsplit_query(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob), key, C.byref(out)))
    return out.value


def query_many(blob: bytes, keys) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.zeros(len(keys), dtype=np.uint64)
    buf = np.frombuffer(blob, dtype=np.uint8)
    _check(lib().recsplit_query_many(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob), _p64(keys),
                                     len(keys), _p64(out)))
    return out


def query_device(blob: bytes, keys_tensor, stream=None):
    """Evaluate on a CUDA tensor of keys on the GPU; returns an int64 CUDA tensor."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(keys_tensor.device)
    out = torch.empty_like(keys_tensor)
    buf = np.frombuffer(blob, dtype=np.uint8)
    _check(lib().recsplit_query_device(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob),
                                       C.c_void_p(keys_tensor.data_ptr()), keys_tensor.numel(),
                                       C.c_void_p(out.data_ptr()), C.c_void_p(stream.cuda_stream)))
    return out


def check_bijective_device(values_tensor, stream=None) -> int:
    """Number of entries of a CUDA tensor outside [0, n) or repeated (0 <=> permutation)."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(values_tensor.device)
    bad = np.zeros(1, dtype=np.uint64)
    _check(lib().recsplit_check_bijective_device(C.c_void_p(values_tensor.data_ptr()), values_tensor.numel(),
                                                 _p64(bad), C.c_void_p(stream.cuda_stream)))
    return int(bad[0])


class Handle:
    """An opened MPHF (recsplit_open): parsed once; with device >= 0 also resident in that
    GPU's HBM for query_device.  Use as a context manager or call close()."""

    def __init__(self, blob: bytes, device: int = -1):
        self._h = C.c_void_p()
        buf = np.frombuffer(blob, dtype=np.uint8)
        _check(lib().recsplit_open(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob), device, C.byref(self._h)))
        self.device = device

    def query_many(self, keys) -> np.ndarray:
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.zeros(len(keys), dtype=np.uint64)
        _check(lib().recsplit_handle_query_many(self._h, _p64(keys), len(keys), _p64(out)))
        return out

    def query_device(self, keys_tensor, out=None, stream=None):
        """Enqueue the GPU query of a CUDA tensor of keys on `stream` (default: the current
        stream); returns the int64 output tensor without synchronising."""
        import torch

        if stream is None:
            stream = torch.cuda.current_stream(keys_tensor.device)
        if out is None:
            out = torch.empty_like(keys_tensor)
        _check(lib().recsplit_handle_query_device(self._h, C.c_void_p(keys_tensor.data_ptr()), keys_tensor.numel(),
                                                  C.c_void_p(out.data_ptr()), C.c_void_p(stream.cuda_stream)))
        return out

    def close(self):
        if self._h:
            lib().recsplit_close(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bits_per_key(blob: bytes) -> float:
    out = C.c_double()
    buf = np.frombuffer(blob, dtype=np.uint8)
    _check(lib().recsplit_bits_per_key(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob), C.byref(out)))
    return out.value


def search_leaves(lo, isb, offsets, rotation_fitting: bool = True) -> np.ndarray:
    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    isb = np.ascontiguousarray(isb, dtype=np.uint8)
    off = np.ascontiguousarray(offsets, dtype=np.uint32)
    out = np.zeros(max(len(off) - 1, 0), dtype=np.uint64)
    _check(lib().recsplit_search_leaves(_p64(lo), isb.ctypes.data_as(C.POINTER(C.c_uint8)),
                                        off.ctypes.data_as(C.POINTER(C.c_uint32)), len(out),
                                        int(rotation_fitting), _p64(out)))
    return out


def search_splits(lo, offsets, leaf_size: int) -> np.ndarray:
    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    off = np.ascontiguousarray(offsets, dtype=np.uint32)
    out = np.zeros(max(len(off) - 1, 0), dtype=np.uint64)
    _check(lib().recsplit_search_splits(_p64(lo), off.ctypes.data_as(C.POINTER(C.c_uint32)), len(out),
                                        leaf_size, _p64(out)))
    return out


def tau(leaf_size: int, s: int, rotation_fitting: bool = True) -> int:
    return _check(lib().recsplit_tau(leaf_size, s, int(rotation_fitting)))


# ---------------------------------------------------------------- sharded builds --

class Shard:
    """One rank's share of a sharded build (include/recsplit.h, recsplit_shard_*)."""

    def __init__(self, keys_tensor, leaf_size: int, bucket_size: int, rank: int, world: int,
                 rotation_fitting: bool = True, global_seed: int = 0, stream=None, total_keys: int = 0,
                 cuts=None):
        """keys_tensor: all keys (total_keys = 0), or exactly the keys this rank owns after
        route_keys + all-to-all (total_keys = the whole build's key count)."""
        import torch

        if not keys_tensor.is_cuda or not keys_tensor.is_contiguous() or keys_tensor.element_size() != 8:
            raise ValueError("keys_tensor must be a contiguous 8-byte CUDA tensor")
        if stream is None:
            stream = torch.cuda.current_stream(keys_tensor.device)
        self._h = C.c_void_p()
        self.summary = np.zeros(8, dtype=np.uint64)
        cuts = None if cuts is None else np.ascontiguousarray(cuts, dtype=np.uint64)
        o = _opts(rotation_fitting, global_seed, keys_tensor.device.index, 0, total_keys, cuts)
        _check(lib().recsplit_shard_begin(C.c_void_p(keys_tensor.data_ptr()), keys_tensor.numel(), leaf_size,
                                          bucket_size, C.byref(o), rank, world, C.c_void_p(stream.cuda_stream),
                                          C.byref(self._h), _p64(self.summary)))

    def min_step(self, summaries: np.ndarray) -> int:
        s = np.ascontiguousarray(summaries, dtype=np.uint64).reshape(-1)
        out = C.c_int64()
        _check(lib().recsplit_shard_min_step(self._h, _p64(s), C.byref(out)))
        return out.value

    def finish(self, min_step: int) -> bytes:
        b = Bytes()
        _check(lib().recsplit_shard_finish(self._h, min_step, C.byref(b)))
        return _take(b)

    def close(self):
        if self._h:
            lib().recsplit_shard_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stitch(parts) -> bytes:
    """Serialized MPHF from the parts of ranks 0..W-1 (host)."""
    bufs = [np.frombuffer(p, dtype=np.uint8) for p in parts]
    ptrs = (C.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    sizes = (C.c_size_t * len(bufs))(*[len(b) for b in bufs])
    out = Bytes()
    _check(lib().recsplit_stitch(ptrs, sizes, len(bufs), C.byref(out)))
    return _take(out)


def shard_globals(summaries, world: int, rank: int) -> dict:
    s = np.ascontiguousarray(summaries, dtype=np.uint64).reshape(-1)
    out = np.zeros(6, dtype=np.uint64)
    _check(lib().recsplit_shard_globals(_p64(s), world, rank, _p64(out)))
    return dict(zip(("n", "D", "delta_C", "beta", "key_base", "bit_base"), (int(x) for x in out)))


def exchange_summaries(summary: np.ndarray, group=None) -> np.ndarray:
    """allgather of the 8-word summaries over torch.distributed (NCCL or gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.from_numpy(summary.view(np.int64).copy()).to(dev)
    out = torch.empty(world * 8, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.cpu().numpy().view(np.uint64).reshape(world, 8)


def allreduce_min(x: int, group=None) -> int:
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


def gather_parts(part: bytes, dst: int = 0, group=None):
    """Variable-length byte parts to rank dst only (list on dst, None elsewhere): the sizes
    are all-gathered (one u64 per rank), the padded parts gathered to dst."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    n = torch.tensor([len(part)], dtype=torch.int64, device=dev)
    sizes = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, n, group=group)
    sizes = sizes.cpu().tolist()
    mx = max(sizes)
    buf = torch.zeros(mx, dtype=torch.uint8)
    buf[:len(part)] = torch.frombuffer(bytearray(part), dtype=torch.uint8)
    buf = buf.to(dev)
    me = dist.get_rank(group)
    dst_g = dist.get_global_rank(group, dst) if group is not None else dst
    if me != dst:
        dist.gather(buf, None, dst=dst_g, group=group)
        return None
    outs = [torch.empty(mx, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.gather(buf, outs, dst=dst_g, group=group)
    return [outs[r][:sizes[r]].cpu().numpy().tobytes() for r in range(world)]


def bucket_histogram(keys_tensor, total_keys: int, bucket_size: int, global_seed: int = 0, stream=None,
                     out=None):
    """Per-global-bucket key counts of this rank's CUDA keys (int32 CUDA tensor of B)."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(keys_tensor.device)
    B = (total_keys + bucket_size - 1) // bucket_size
    if out is None:
        out = torch.zeros(B, dtype=torch.int32, device=keys_tensor.device)
    o = _opts(True, global_seed, keys_tensor.device.index, 0)
    _check(lib().recsplit_bucket_histogram(C.c_void_p(keys_tensor.data_ptr()), keys_tensor.numel(), total_keys,
                                           bucket_size, C.byref(o), C.c_void_p(stream.cuda_stream),
                                           C.c_void_p(out.data_ptr())))
    return out


def balanced_cuts(hist, leaf_size: int, world: int, rotation_fitting: bool = True) -> np.ndarray:
    """world + 1 bucket cuts with about equal expected work (recsplit_balanced_cuts)."""
    h = np.ascontiguousarray(hist, dtype=np.uint32)
    cuts = np.zeros(world + 1, dtype=np.uint64)
    _check(lib().recsplit_balanced_cuts(h.ctypes.data_as(C.POINTER(C.c_uint32)), len(h), leaf_size,
                                        int(rotation_fitting), world, _p64(cuts)))
    return cuts


def route_keys(keys_tensor, total_keys: int, bucket_size: int, world: int, global_seed: int = 0, stream=None,
               cuts=None):
    """Group this rank's CUDA keys by the rank that owns their bucket (recsplit_route_keys):
    returns (keys grouped rank by rank, list of per-rank counts)."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(keys_tensor.device)
    out = torch.empty_like(keys_tensor)
    counts = np.zeros(world, dtype=np.uint64)
    cuts = None if cuts is None else np.ascontiguousarray(cuts, dtype=np.uint64)
    o = _opts(True, global_seed, keys_tensor.device.index, 0, cuts=cuts)
    _check(lib().recsplit_route_keys(C.c_void_p(keys_tensor.data_ptr()), keys_tensor.numel(), total_keys,
                                     bucket_size, C.byref(o), world, C.c_void_p(stream.cuda_stream),
                                     C.c_void_p(out.data_ptr()), _p64(counts)))
    return out, [int(c) for c in counts]


def exchange_keys(routed, send_counts, group=None):
    """all-to-all of routed keys (NCCL: device buffers; gloo: through host memory): returns
    the keys this rank owns, on routed's device."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = routed.device if nccl else torch.device("cpu")
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = rc.cpu().tolist()
    src = routed if nccl else routed.cpu()
    recv = torch.empty(sum(recv_counts), dtype=routed.dtype, device=dev)
    dist.all_to_all_single(recv, src, output_split_sizes=recv_counts, input_split_sizes=list(send_counts),
                           group=group)
    return recv if nccl else recv.to(routed.device)


def allreduce_sum(x: int, group=None) -> int:
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def global_histogram(keys_tensor, total_keys: int, bucket_size: int, global_seed: int = 0, group=None,
                     stream=None, distributed: bool = True) -> np.ndarray:
    """Bucket sizes of the whole build (B entries, host): this rank's histogram, summed over
    the group when each rank holds a slice (distributed=True, one allreduce of B int32)."""
    import torch.distributed as dist

    h = bucket_histogram(keys_tensor, total_keys, bucket_size, global_seed, stream)
    if distributed and dist.get_world_size(group) > 1:
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(h, group=group)
        else:
            hc = h.cpu()
            dist.all_reduce(hc, group=group)
            h = hc
    return h.cpu().numpy().astype(np.uint32)


def build_sharded(keys_tensor, leaf_size: int, bucket_size: int, rotation_fitting: bool = True,
                  global_seed: int = 0, group=None, stream=None, distribute: bool = False, balance: bool = True):
    """Multi-GPU build of ONE MPHF over the torch.distributed group (one rank per GPU):
    bucket ranges per rank, allgather of summaries, allreduce-min of the residual step,
    parts gathered to rank 0 and stitched.  Returns the bytes on rank 0, None elsewhere.
    distribute=False: every rank passes ALL keys (each keeps its buckets);
    distribute=True: each rank passes its own slice of the input; the keys are routed to
    their owners with one all-to-all.
    balance=True: contiguous bucket ranges of about equal expected work (bucket-size
    histogram -> recsplit_balanced_cuts; one extra allreduce of B int32 when distributed);
    False: equal bucket counts.  The output bytes are the same either way."""
    import os
    import time

    import torch.distributed as dist

    trace = os.environ.get("RS_TRACE_SHARDED")  # (development: stage wall times to stderr)
    marks = [("start", time.perf_counter())]

    def mark(name):
        if trace:
            marks.append((name, time.perf_counter()))

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    total = allreduce_sum(keys_tensor.numel(), group) if distribute else keys_tensor.numel()
    cuts = None
    if balance and world > 1:
        hist = global_histogram(keys_tensor, total, bucket_size, global_seed, group, stream, distribute)
        mark("histogram")
        cuts = balanced_cuts(hist, leaf_size, world, rotation_fitting)
        mark("cuts")
    if distribute:
        routed, counts = route_keys(keys_tensor, total, bucket_size, world, global_seed, stream, cuts)
        mark("route")
        keys_tensor = exchange_keys(routed, counts, group)
        mark("exchange")
        del routed
    sh = Shard(keys_tensor, leaf_size, bucket_size, rank, world, rotation_fitting, global_seed, stream,
               total if distribute else 0, cuts)
    mark("shard")
    try:
        allsum = exchange_summaries(sh.summary, group)
        step = allreduce_min(sh.min_step(allsum), group)
        part = sh.finish(step)
        mark("finish")
    finally:
        sh.close()
    parts = gather_parts(part, 0, group)
    mark("gather")
    out = stitch(parts) if parts is not None else None
    mark("stitch")
    if trace:
        import sys
        print(f"[rank {rank}] build_sharded ms: " + ", ".join(
            f"{n} {1e3 * (t - marks[i][1]):.2f}" for i, (n, t) in enumerate(marks[1:])), file=sys.stderr, flush=True)
    return out


def trim() -> None:
    """Release the library's cached build graphs and workspaces, unused pool memory and idle
    pinned buffers (recsplit_trim)."""
    _check(lib().recsplit_trim())
