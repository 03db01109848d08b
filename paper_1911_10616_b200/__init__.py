"""B200-native EVOKE: n x 73 vertex-orbit counts for all connected 2..5-vertex patterns.

Thin Python binding over the C ABI in ``include/evoke.h`` (``libevoke.so`` built from
``csrc/`` for sm_100a).  This module only marshals arguments: every step of the counted
method runs in the CUDA kernels of the library.  There is no CPU fallback -- if the
shared library is missing the import of a binding function raises.

    evoke_orbits_edges(n, edges, ...)   -> uint64[n, 73]
    evoke_orbits_csr(n, rowptr, col, ...) -> uint64[n, 73]

Inputs may be numpy arrays (host pointers; the library copies them to the GPU inside the
call) or CUDA torch tensors (device pointers; no host transfer).  ``num_shards`` /
``shard_index`` select a data-parallel shard: the element-wise sum (mod 2^64) of the
partial matrices of all shards equals the full result (see ``parallel.py``).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

NUM_ORBITS = 73
_HERE = os.path.dirname(os.path.abspath(__file__))
# (EVOKE_LIB_PATH: developer A/B of two builds of the library; default the in-tree build)
LIB_PATH = os.environ.get("EVOKE_LIB_PATH") or os.path.join(_HERE, "libevoke.so")

EVOKE_OK, EVOKE_EINVAL, EVOKE_ENOMEM, EVOKE_ECUDA, EVOKE_EINTERNAL = 0, -1, -2, -3, -5


class EvokeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"evoke error {code}: {msg}")
        self.code = code


class _Stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("triangles", ctypes.c_int64),
                ("max_degree", ctypes.c_int64), ("degeneracy", ctypes.c_int64), ("wedges", ctypes.c_int64),
                ("ms_total", ctypes.c_double), ("ms_pass", ctypes.c_double * 16),
                ("num_passes", ctypes.c_int32), ("kernel_launches", ctypes.c_int32),
                ("library_launches", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("alg_bytes", ctypes.c_double * 16), ("units", ctypes.c_int64 * 8),
                ("work_shard", ctypes.c_uint64 * 4), ("work_total", ctypes.c_uint64 * 4)]


class _Options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("induced", ctypes.c_int32),
                ("device_pointers", ctypes.c_int32), ("shard_index", ctypes.c_int32),
                ("num_shards", ctypes.c_int32), ("device", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("stats", ctypes.POINTER(_Stats))]

SHARDED_PASSES = ("pair_pass", "hub_local", "cycles5", "cliques")
FLAG_WORKMODEL = 1
FLAG_SERIAL = 2
FLAG_FOUR = 4


_lock = threading.Lock()
_lib = None

EXPORTED_SYMBOLS = ("evoke_default_options", "evoke_orbits_edges", "evoke_orbits_csr", "evoke_pass_name",
                    "evoke_strerror", "evoke_last_error", "evoke_version", "evoke_ccd", "evoke_release_scratch",
                    "evoke_orbits_edges_multi")


def lib():
    """Load libevoke.so (raises if it has not been built -- no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                                  f"g.build()'` (nvcc, sm_100a)")
            L = ctypes.CDLL(LIB_PATH)
            L.evoke_default_options.argtypes = [ctypes.POINTER(_Options)]
            L.evoke_orbits_edges.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.POINTER(_Options)]
            L.evoke_orbits_edges.restype = ctypes.c_int
            L.evoke_orbits_csr.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.POINTER(_Options)]
            L.evoke_orbits_csr.restype = ctypes.c_int
            L.evoke_orbits_edges_multi.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                                   ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                                   ctypes.POINTER(_Options)]
            L.evoke_orbits_edges_multi.restype = ctypes.c_int
            L.evoke_ccd.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(_Options)]
            L.evoke_ccd.restype = ctypes.c_int
            for f in ("evoke_pass_name",):
                getattr(L, f).argtypes = [ctypes.c_int]
                getattr(L, f).restype = ctypes.c_char_p
            L.evoke_strerror.argtypes = [ctypes.c_int]
            L.evoke_strerror.restype = ctypes.c_char_p
            L.evoke_last_error.restype = ctypes.c_char_p
            L.evoke_version.restype = ctypes.c_char_p
            L.evoke_release_scratch.argtypes = [ctypes.c_int]
            L.evoke_release_scratch.restype = ctypes.c_int
            _lib = L
    return _lib


def version() -> str:
    return lib().evoke_version().decode()


def evoke_release_scratch(device: int = -1) -> None:
    """Free the zeroed per-device scratch the library keeps between calls (-1: all devices)."""
    _check(lib().evoke_release_scratch(int(device)))


def pass_names() -> list[str]:
    L = lib()
    out = []
    i = 0
    while True:
        s = L.evoke_pass_name(i)
        if s is None:
            break
        out.append(s.decode())
        i += 1
    return out


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _make_options(induced, device_pointers, shard_index, num_shards, device, stream, stats, flags=0):
    o = _Options()
    lib().evoke_default_options(ctypes.byref(o))
    o.flags = flags
    o.induced = 1 if induced else 0
    o.device_pointers = 1 if device_pointers else 0
    o.shard_index = shard_index
    o.num_shards = num_shards
    o.device = -1 if device is None else int(device)
    o.stream = stream
    o.stats = ctypes.pointer(stats) if stats is not None else None
    return o


def _stats_dict(s: _Stats) -> dict:
    names = pass_names()
    return {"n": s.n, "m": s.m, "triangles": s.triangles, "max_degree": s.max_degree,
            "degeneracy": s.degeneracy, "wedges": s.wedges, "ms_total": s.ms_total,
            "ms_pass": {names[i]: s.ms_pass[i] for i in range(min(s.num_passes, len(names)))},
            "alg_bytes": {names[i]: s.alg_bytes[i] for i in range(min(s.num_passes, len(names)))},
            "units": {k: s.units[i] for i, k in enumerate(("sum_d2", "sum_te2", "hub", "c5_wedge", "c5_q",
                                                           "tri_stream", "pair_rwedge", "pair_hwalk"))},
            "kernel_launches": s.kernel_launches, "library_launches": s.library_launches,
            "work_shard": {k: s.work_shard[i] for i, k in enumerate(SHARDED_PASSES)},
            "work_total": {k: s.work_total[i] for i, k in enumerate(SHARDED_PASSES)}}


def _check(rc: int):
    if rc != EVOKE_OK:
        L = lib()
        raise EvokeError(rc, f"{L.evoke_strerror(rc).decode()}: {L.evoke_last_error().decode()}")


def evoke_orbits_edges(n: int, edges, out=None, induced: bool = True, shard_index: int = 0,
                       num_shards: int = 1, stream=None, return_stats: bool = False, workmodel: bool = False,
                       serial: bool = False, four_only: bool = False):
    """Orbit counts uint64[n, 73] of the simple graph given by undirected pairs ``edges``.

    ``edges``: int32 [m, 2] numpy array (host) or CUDA torch tensor (device).  Duplicates,
    reverse duplicates and self-loops are removed by the library.
    ``out``: optional preallocated numpy uint64 [n, 73] (host input) or torch int64/uint64
    CUDA tensor [n, 73] (device input)."""
    st = _Stats() if (return_stats or workmodel) else None
    fl = (FLAG_WORKMODEL if workmodel else 0) | (FLAG_SERIAL if serial else 0) | (FLAG_FOUR if four_only else 0)
    if _is_torch(edges):
        import torch
        assert edges.is_cuda and edges.dtype == torch.int32, "device edges must be CUDA int32"
        e = edges.contiguous()
        m = e.numel() // 2
        if out is None:
            out = torch.empty((n, NUM_ORBITS), dtype=torch.int64, device=e.device)
        assert out.is_cuda and out.device == e.device and out.is_contiguous() and out.numel() == n * NUM_ORBITS
        if stream is None:
            stream = torch.cuda.current_stream(e.device).cuda_stream
        o = _make_options(induced, True, shard_index, num_shards, e.device.index, stream, st, fl)
        rc = lib().evoke_orbits_edges(n, m, e.data_ptr(), out.data_ptr(), ctypes.byref(o))
    else:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
        m = e.shape[0]
        if out is None:
            out = np.zeros((n, NUM_ORBITS), dtype=np.uint64)
        assert out.dtype == np.uint64 and out.flags.c_contiguous and out.size == n * NUM_ORBITS
        o = _make_options(induced, False, shard_index, num_shards, None, stream, st, fl)
        rc = lib().evoke_orbits_edges(n, m, e.ctypes.data if m else None, out.ctypes.data, ctypes.byref(o))
    _check(rc)
    if return_stats or workmodel:
        return out, _stats_dict(st)
    return out


def evoke_orbits_edges_multi(n: int, edges, devices, out=None, induced: bool = True, shard_index: int = 0,
                             num_shards: int = 1, return_stats: bool = False, four_only: bool = False):
    """The same matrix computed on several GPUs of this process (C ABI
    ``evoke_orbits_edges_multi``): shard d of len(devices) runs on devices[d], devices[0]
    sums the partials over peer memory.  ``edges``: numpy int32 [m, 2] (host) or a CUDA torch
    tensor on devices[0]; ``out`` as for ``evoke_orbits_edges``."""
    st = _Stats() if return_stats else None
    fl = FLAG_FOUR if four_only else 0
    devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
    if _is_torch(edges):
        import torch
        assert edges.is_cuda and edges.dtype == torch.int32, "device edges must be CUDA int32"
        assert edges.device.index == int(devices[0]), "device edges must live on devices[0]"
        e = edges.contiguous()
        m = e.numel() // 2
        if out is None:
            out = torch.empty((n, NUM_ORBITS), dtype=torch.int64, device=e.device)
        assert out.is_cuda and out.device == e.device and out.is_contiguous() and out.numel() == n * NUM_ORBITS
        torch.cuda.synchronize(e.device)  # the library's per-device streams do not see torch's
        o = _make_options(induced, True, shard_index, num_shards, None, None, st, fl)
        rc = lib().evoke_orbits_edges_multi(n, m, e.data_ptr(), out.data_ptr(), devs, len(devices), ctypes.byref(o))
    else:
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
        m = e.shape[0]
        if out is None:
            out = np.zeros((n, NUM_ORBITS), dtype=np.uint64)
        assert out.dtype == np.uint64 and out.flags.c_contiguous and out.size == n * NUM_ORBITS
        o = _make_options(induced, False, shard_index, num_shards, None, None, st, fl)
        rc = lib().evoke_orbits_edges_multi(n, m, e.ctypes.data if m else None, out.ctypes.data, devs, len(devices),
                                            ctypes.byref(o))
    _check(rc)
    if return_stats:
        return out, _stats_dict(st)
    return out


def evoke_orbits_csr(n: int, rowptr, col, out=None, induced: bool = True, shard_index: int = 0,
                     num_shards: int = 1, stream=None, return_stats: bool = False, workmodel: bool = False,
                     serial: bool = False, four_only: bool = False):
    """Orbit counts from a CSR (rowptr int64[n+1], col int32[rowptr[n]]); same cleaning."""
    st = _Stats() if (return_stats or workmodel) else None
    fl = (FLAG_WORKMODEL if workmodel else 0) | (FLAG_SERIAL if serial else 0) | (FLAG_FOUR if four_only else 0)
    if _is_torch(rowptr):
        import torch
        assert rowptr.is_cuda and rowptr.dtype == torch.int64, "device rowptr must be CUDA int64"
        assert col.is_cuda and col.dtype == torch.int32, "device col must be CUDA int32"
        assert rowptr.device == col.device and rowptr.numel() == n + 1
        rp = rowptr.contiguous()
        cl = col.contiguous()
        if out is None:
            out = torch.empty((n, NUM_ORBITS), dtype=torch.int64, device=rp.device)
        assert out.is_cuda and out.device == rp.device and out.is_contiguous() and out.numel() == n * NUM_ORBITS
        if stream is None:
            stream = torch.cuda.current_stream(rp.device).cuda_stream
        o = _make_options(induced, True, shard_index, num_shards, rp.device.index, stream, st, fl)
        rc = lib().evoke_orbits_csr(n, rp.data_ptr(), cl.data_ptr(), out.data_ptr(), ctypes.byref(o))
    else:
        rp = np.ascontiguousarray(np.asarray(rowptr, dtype=np.int64))
        cl = np.ascontiguousarray(np.asarray(col, dtype=np.int32))
        assert rp.size == n + 1, "rowptr must have n + 1 entries"
        if out is None:
            out = np.zeros((n, NUM_ORBITS), dtype=np.uint64)
        assert out.dtype == np.uint64 and out.flags.c_contiguous and out.size == n * NUM_ORBITS
        o = _make_options(induced, False, shard_index, num_shards, None, stream, st, fl)
        rc = lib().evoke_orbits_csr(n, rp.ctypes.data, cl.ctypes.data if cl.size else None, out.ctypes.data,
                                    ctypes.byref(o))
    _check(rc)
    if return_stats or workmodel:
        return out, _stats_dict(st)
    return out


def evoke_ccd(dim, orbit: int):
    """Complementary cumulative distribution of orbit column ``orbit`` of an orbit matrix
    ``dim`` (numpy uint64 [n, 73]): returns (values, counts), values ascending distinct
    counts, counts[i] = number of vertices whose count is >= values[i]."""
    d = np.ascontiguousarray(dim).view(np.uint64)
    n = d.shape[0]
    values = np.zeros(max(n, 1), dtype=np.uint64)
    counts = np.zeros(max(n, 1), dtype=np.uint64)
    k = ctypes.c_int64(0)
    o = _make_options(True, False, 0, 1, None, None, None, 0)
    rc = lib().evoke_ccd(n, d.ctypes.data if n else None, int(orbit), values.ctypes.data, counts.ctypes.data,
                         ctypes.byref(k), ctypes.byref(o))
    _check(rc)
    return values[:k.value], counts[:k.value]
