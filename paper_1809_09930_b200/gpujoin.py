"""Thin ctypes binding of libgpujoin.so (include/gpujoin.h).  Argument
marshalling only: every step of the self-join runs in the CUDA library.  The
functions keep the C names without the ``gj_`` prefix.

Loading fails loudly when the library has not been built; there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgpujoin.so")

GJ_OK, GJ_ERR_INVALID, GJ_ERR_CUDA, GJ_ERR_OVERFLOW, GJ_ERR_CAPACITY, GJ_ERR_NOMEM = 0, -1, -2, -3, -4, -5

# Every symbol include/gpujoin.h declares (checked by tests/test_capi_cpu.py).
EXPORTS = ["gj_default_options", "gj_build_index", "gj_index_info", "gj_dim_order", "gj_device_arrays",
           "gj_estimate", "gj_num_batches", "gj_partition", "gj_fp32_threshold", "gj_fp32_accept_threshold", "gj_tc_threshold", "gj_selftest_umma", "gj_self_join_async", "gj_self_join_async_stream", "gj_self_join_count_async", "gj_self_join",
           "gj_self_join_host", "gj_join_stats", "gj_join_counts", "gj_join_mma_tests", "gj_neighbor_table", "gj_free_index", "gj_last_error",
           "gj_abi_version", "gj_launch_count", "gj_release_cached_memory"]


class Options(C.Structure):
    _fields_ = [("reorder", C.c_int32), ("sortidu", C.c_int32), ("shortc", C.c_int32), ("symmetric", C.c_int32),
                ("sample_frac", C.c_double), ("stream", C.c_uint64), ("filter", C.c_int32),
                ("mma_tiles", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("n_points", C.c_int64), ("dim", C.c_int32), ("dim_pad", C.c_int32), ("k", C.c_int32),
                ("u", C.c_int32), ("eps", C.c_double), ("n_cells", C.c_int64), ("n_adjacent", C.c_int64),
                ("n_tiles", C.c_int64), ("est_candidates", C.c_double), ("build_ms", C.c_double),
                ("filter", C.c_int32), ("filter_threshold", C.c_float), ("filter_margin", C.c_double),
                ("tile_queries", C.c_int32), ("mma_depth", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("cells", C.c_int64), ("tests", C.c_int64), ("dims", C.c_int64), ("pairs", C.c_int64),
                ("tests_evaluated", C.c_int64), ("dims_evaluated", C.c_int64)]


class GpuJoinError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gpujoin error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libgpujoin.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, U64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "gj_default_options": (None, [C.POINTER(Options)]),
        "gj_build_index": (C.c_int, [P, I64, I32, D, I32, C.POINTER(Options), C.POINTER(P)]),
        "gj_index_info": (C.c_int, [P, C.POINTER(Info)]),
        "gj_dim_order": (C.c_int, [P, C.POINTER(C.c_int32), I32]),
        "gj_device_arrays": (C.c_int, [P, C.POINTER(P), C.POINTER(P)]),
        "gj_estimate": (C.c_int, [P, D, I32, I32, C.POINTER(I64)]),
        "gj_num_batches": (I64, [I64, I64]),
        "gj_selftest_umma": (C.c_int, [P, P, P, U64]),
        "gj_tc_threshold": (C.c_int, [D, I32, I32, D, D, C.POINTER(D), C.POINTER(D)]),
        "gj_fp32_threshold": (C.c_int, [D, I32, C.POINTER(C.c_double), C.POINTER(C.c_float), C.POINTER(D)]),
        "gj_fp32_accept_threshold": (C.c_int, [D, I32, C.POINTER(C.c_double), C.POINTER(C.c_float)]),
        "gj_partition": (C.c_int, [I64, I32, I32, I32, I32, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64),
                                   C.POINTER(I32)]),
        "gj_self_join_async": (C.c_int, [P, P, I64, P, I32, I32, I32, I32]),
        "gj_self_join_async_stream": (C.c_int, [P, P, I64, P, I32, I32, I32, I32, U64]),
        "gj_self_join_count_async": (C.c_int, [P, P, I32, I32, I32, I32]),
        "gj_self_join": (C.c_int, [P, P, I64, I32, I32, C.POINTER(I64)]),
        "gj_self_join_host": (C.c_int, [P, P, I64, I32, I32, I64, C.POINTER(I64), C.POINTER(C.c_int32)]),
        "gj_join_stats": (C.c_int, [P, I32, I32, C.POINTER(Stats)]),
        "gj_join_counts": (C.c_int, [P, I32, I32, C.POINTER(Stats)]),
        "gj_join_mma_tests": (C.c_int, [P, I32, I32, C.POINTER(I64)]),
        "gj_neighbor_table": (C.c_int, [P, P, I64, P]),
        "gj_free_index": (None, [P]),
        "gj_last_error": (C.c_char_p, []),
        "gj_abi_version": (C.c_int32, []),
        "gj_launch_count": (C.c_int64, []),
        "gj_release_cached_memory": (C.c_int, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc):
    if rc != GJ_OK:
        raise GpuJoinError(rc, lib().gj_last_error().decode())


def default_options(reorder=True, sortidu=True, shortc=True, sample_frac=0.01, stream=0, symmetric=True,
                    filter=2, mma_tiles=0) -> Options:
    o = Options()
    lib().gj_default_options(C.byref(o))
    o.reorder, o.sortidu, o.shortc, o.symmetric = int(reorder), int(sortidu), int(shortc), int(symmetric)
    o.filter = int(filter)
    o.mma_tiles = int(mma_tiles)
    o.sample_frac = float(sample_frac)
    o.stream = int(stream)
    return o


def _ptr(x):
    """Raw pointer of a torch tensor or numpy array (no copies here)."""
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(type(x))


class _CudaView:
    """__cuda_array_interface__ wrapper of a raw device pointer (read-only view)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = dict(shape=tuple(shape), typestr=typestr, data=(int(ptr), False),
                                             version=3, strides=None)


class Index:
    """Handle of gj_build_index.  ``points`` = |D| x n float64, a CUDA torch
    tensor (stays on the device) or a host numpy array / tensor (staged)."""

    def __init__(self, points, eps: float, k: int, reorder=True, sortidu=True, shortc=True, sample_frac=0.01,
                 stream=None, symmetric=True, filter=2, mma_tiles=0):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0
        if isinstance(points, np.ndarray):
            points = np.ascontiguousarray(points, dtype=np.float64)
        else:
            if points.dtype != torch.float64 or not points.is_contiguous():
                raise ValueError("points must be a contiguous float64 tensor")
        self._keep = points
        n, dim = points.shape
        self.n_points, self.dim = int(n), int(dim)
        self.options = default_options(reorder, sortidu, shortc, sample_frac, stream, symmetric, filter, mma_tiles)
        h = C.c_void_p()
        _check(lib().gj_build_index(_ptr(points), n, dim, float(eps), int(k), C.byref(self.options), C.byref(h)))
        self._h = h
        self._keep = None

    # ------------------------------------------------------------------ info
    def info(self) -> Info:
        i = Info()
        _check(lib().gj_index_info(self._h, C.byref(i)))
        return i

    def dim_order(self) -> np.ndarray:
        buf = (C.c_int32 * self.dim)()
        rc = lib().gj_dim_order(self._h, buf, self.dim)
        if rc < 0:
            _check(rc)
        return np.frombuffer(buf, dtype=np.int32).copy()

    def device_arrays(self):
        """(sorted reordered points [N, dim_pad] float64, sorted->original id
        [N] int32) as zero-copy torch views of the index's device memory."""
        import torch
        p, o = C.c_void_p(), C.c_void_p()
        _check(lib().gj_device_arrays(self._h, C.byref(p), C.byref(o)))
        i = self.info()
        pts = torch.as_tensor(_CudaView(p.value, (i.n_points, i.dim_pad), "<f8"), device="cuda")
        ids = torch.as_tensor(_CudaView(o.value, (i.n_points,), "<i4"), device="cuda")
        return pts, ids

    # ------------------------------------------------------------------ join
    def estimate(self, frac=0.01, rank=0, world=1) -> int:
        e = C.c_int64()
        _check(lib().gj_estimate(self._h, float(frac), rank, world, C.byref(e)))
        return e.value

    def self_join_async(self, out_pairs, count, batch=0, n_batches=1, rank=0, world=1, stream=None):
        """Enqueue one batch into device tensors out_pairs (uint32 [cap, 2] as
        int32/uint32 tensor) and count (uint64/int64 device scalar); on the
        index's stream, or on `stream` (a cudaStream_t handle, gj_self_join_async_stream)."""
        cap = out_pairs.shape[0] if out_pairs is not None else 0
        if stream is None:
            _check(lib().gj_self_join_async(self._h, _ptr(out_pairs) if cap else None, cap, _ptr(count), batch,
                                            n_batches, rank, world))
        else:
            _check(lib().gj_self_join_async_stream(self._h, _ptr(out_pairs) if cap else None, cap, _ptr(count),
                                                   batch, n_batches, rank, world, int(stream)))

    def self_join_count_async(self, count, batch=0, n_batches=1, rank=0, world=1):
        _check(lib().gj_self_join_count_async(self._h, _ptr(count), batch, n_batches, rank, world))

    def self_join(self, out_pairs, rank=0, world=1) -> int:
        n = C.c_int64()
        rc = lib().gj_self_join(self._h, _ptr(out_pairs), out_pairs.shape[0], rank, world, C.byref(n))
        if rc == GJ_ERR_CAPACITY:
            raise GpuJoinError(rc, f"capacity {out_pairs.shape[0]} < {n.value} pairs")
        _check(rc)
        return n.value

    def self_join_host(self, out_pairs, rank=0, world=1, batch_size=0):
        """Full pipeline into a host buffer (numpy uint32 [cap,2] or pinned
        torch tensor).  Returns (n_pairs, n_batches)."""
        n, nb = C.c_int64(), C.c_int32()
        rc = lib().gj_self_join_host(self._h, _ptr(out_pairs), out_pairs.shape[0], rank, world, int(batch_size),
                                     C.byref(n), C.byref(nb))
        if rc == GJ_ERR_CAPACITY:
            raise GpuJoinError(rc, f"capacity {out_pairs.shape[0]} < {n.value} pairs")
        _check(rc)
        return n.value, nb.value

    def stats(self, rank=0, world=1) -> dict:
        s = Stats()
        _check(lib().gj_join_stats(self._h, rank, world, C.byref(s)))
        return dict(cells=s.cells, tests=s.tests, dims=s.dims, pairs=s.pairs, tests_evaluated=s.tests_evaluated,
                    dims_evaluated=s.dims_evaluated)

    def counts(self, rank=0, world=1) -> dict:
        """cells / tests / tests_evaluated without the distance work (gj_join_counts)."""
        s = Stats()
        _check(lib().gj_join_counts(self._h, rank, world, C.byref(s)))
        return dict(cells=s.cells, tests=s.tests, tests_evaluated=s.tests_evaluated)

    def mma_tests(self, rank=0, world=1) -> int:
        """Executed tensor-core accumulator entries of the share (gj_join_mma_tests; -1 if not filter 2)."""
        v = C.c_int64(0)
        _check(lib().gj_join_mma_tests(self._h, rank, world, C.byref(v)))
        return int(v.value)

    def neighbor_table(self, pairs, n_pairs, offsets):
        _check(lib().gj_neighbor_table(self._h, _ptr(pairs), int(n_pairs), _ptr(offsets)))

    def free(self):
        if getattr(self, "_h", None):
            lib().gj_free_index(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def num_batches(est_pairs: int, batch_size: int) -> int:
    return int(lib().gj_num_batches(int(est_pairs), int(batch_size)))


def partition(n_tiles: int, rank: int, world: int, batch: int = 0, n_batches: int = 1):
    """(first, step, count, block) of (rank, batch) -- gj_partition: query sets
    first + step * k of `block` consecutive tile positions, count positions."""
    f, s, c, b = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
    _check(lib().gj_partition(int(n_tiles), rank, world, batch, n_batches, C.byref(f), C.byref(s), C.byref(c),
                              C.byref(b)))
    return f.value, s.value, c.value, b.value


def fp32_threshold(eps: float, spans):
    """(enabled, threshold float32, margin) of the certified FP32 prefilter."""
    sp = np.ascontiguousarray(spans, dtype=np.float64)
    t, m = C.c_float(), C.c_double()
    rc = lib().gj_fp32_threshold(float(eps), len(sp), sp.ctypes.data_as(C.POINTER(C.c_double)), C.byref(t),
                                 C.byref(m))
    if rc < 0:
        _check(rc)
    return bool(rc), np.float32(t.value), m.value


def fp32_accept_threshold(eps: float, spans):
    """Certain-inside float32 threshold of the FP32 filter (-1: none)."""
    sp = np.ascontiguousarray(spans, dtype=np.float64)
    t = C.c_float()
    _check(lib().gj_fp32_accept_threshold(float(eps), len(sp), sp.ctypes.data_as(C.POINTER(C.c_double)), C.byref(t)))
    return np.float32(t.value)


def tc_threshold(eps: float, n: int, K: int, S: float, R2: float):
    """(enabled, T, margin) of the certified tensor-core bound (gj_tc_threshold)."""
    t, m = C.c_double(), C.c_double()
    rc = lib().gj_tc_threshold(float(eps), int(n), int(K), float(S), float(R2), C.byref(t), C.byref(m))
    if rc < 0:
        _check(rc)
    return bool(rc), t.value, m.value


def selftest_umma(A, B, D, stream=0):
    """tcgen05 self-test GEMM: D[128,128] = A[128,32] @ B[128,32]^T (fp16 in, fp32 out, CUDA tensors)."""
    _check(lib().gj_selftest_umma(_ptr(A), _ptr(B), _ptr(D), int(stream)))


def launch_count() -> int:
    """Kernels launched by libgpujoin in this process so far."""
    return int(lib().gj_launch_count())


def release_cached_memory() -> None:
    """Return the library pool's cached device memory to the driver (gj_release_cached_memory)."""
    _check(lib().gj_release_cached_memory())


def abi_version() -> int:
    return int(lib().gj_abi_version())
