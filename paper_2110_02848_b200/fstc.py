"""Thin ctypes binding of libfstc (include/fstc.h) -- argument marshalling only.

Every step of composition runs in the CUDA kernels of libfstc.so; this module only converts
numpy arrays / torch tensors into the C descriptors and back.  There is no CPU fallback: if the
library is missing or no CUDA device is usable, every call raises ``FstError``.

Names mirror the C ABI: fst_create, fst_compose, fst_compose_batch, fst_free, fst_info,
fst_copy_to_host, fst_get_stats, fst_level_sizes, fst_adjacency.  ``Fst`` is a small owning
wrapper around a handle.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSTC_LIB") or os.path.join(_HERE, "libfstc.so")  # FSTC_LIB: A/B runs (scripts/ab_build.sh)

FST_EPS = -1
FST_MEM_DEVICE, FST_MEM_HOST = 0, 1
STATUS = {0: "FST_OK", 1: "FST_E_INVALID_ARG", 2: "FST_E_INVALID_GRAPH", 3: "FST_E_OOM", 4: "FST_E_CAPACITY",
          5: "FST_E_CUDA", 6: "FST_E_NCCL", 7: "FST_E_INTERNAL"}

EXPORTED = ["fst_create", "fst_compose", "fst_compose_batch", "fst_free", "fst_info", "fst_copy_to_host",
            "fst_get_stats", "fst_level_sizes", "fst_adjacency", "fst_set_profiling", "fst_set_tile_mode", "fst_set_wave_mode", "fst_launch_count",
            "fst_last_error", "fst_version", "fst_comm_unique_id", "fst_comm_init", "fst_comm_destroy",
            "fst_compose_sharded", "fst_compose_sharded_local", "fst_shard_info", "fst_copy_arcs_to_host",
            "fst_compose_ex", "fst_compose_batch_ex", "fst_copy_provenance_to_host", "fst_grad_scatter",
            "fst_forward_score", "fst_copy_pair_f_to_host", "fst_compose_chain"]
FST_COMPOSE_PROVENANCE = 1
FST_COMPOSE_EPS_FILTER = 2


class FstError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class fst_desc(C.Structure):
    _fields_ = [("num_states", C.c_int32), ("num_arcs", C.c_int64), ("row_ptr", C.c_void_p),
                ("ilabel", C.c_void_p), ("olabel", C.c_void_p), ("dst", C.c_void_p), ("weight", C.c_void_p),
                ("is_start", C.c_void_p), ("is_accept", C.c_void_p), ("memory", C.c_int32)]


class fst_view(C.Structure):
    _fields_ = [("num_states", C.c_int32), ("num_arcs", C.c_int64), ("row_ptr", C.c_void_p),
                ("ilabel", C.c_void_p), ("olabel", C.c_void_p), ("dst", C.c_void_p), ("weight", C.c_void_p),
                ("is_start", C.c_void_p), ("is_accept", C.c_void_p), ("pair_a", C.c_void_p),
                ("pair_b", C.c_void_p), ("arc_a", C.c_void_p), ("arc_b", C.c_void_p), ("pair_f", C.c_void_p)]


class fst_compose_stats(C.Structure):
    _fields_ = [("levels_stage1", C.c_int32), ("levels_stage2", C.c_int32), ("num_coaccessible", C.c_int64),
                ("pair_space", C.c_int64), ("ms_stage1", C.c_float), ("ms_stage2", C.c_float),
                ("ms_number", C.c_float), ("ms_alloc", C.c_float), ("ms_emit", C.c_float),
                ("ms_total", C.c_float), ("launches", C.c_int64), ("emit_launches", C.c_int64),
                ("expand_launches", C.c_int64), ("staged_tasks", C.c_int64), ("tile_path", C.c_int32),
                ("pull_levels", C.c_int32), ("ms_count", C.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class fst_shard_desc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("state_offset", C.c_int64), ("arc_offset", C.c_int64),
                ("total_states", C.c_int64), ("total_arcs", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads libfstc.so (built by ``__graft_entry__.build()``); raises if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise FstError(5, f"{path} not built -- run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(path)
        vp = C.c_void_p
        lib.fst_create.argtypes = [C.POINTER(fst_desc), vp, C.POINTER(vp)]
        lib.fst_compose.argtypes = [vp, vp, vp, C.POINTER(vp)]
        lib.fst_compose_batch.argtypes = [C.c_int32, C.POINTER(vp), C.POINTER(vp), vp, C.POINTER(vp)]
        lib.fst_free.argtypes = [vp]
        lib.fst_free.restype = None
        lib.fst_info.argtypes = [vp, C.POINTER(fst_view)]
        lib.fst_copy_to_host.argtypes = [vp, vp] + [vp] * 9
        lib.fst_get_stats.argtypes = [vp, C.POINTER(fst_compose_stats)]
        lib.fst_copy_arcs_to_host.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, vp, vp, vp]
        if hasattr(lib, "fst_compose_ex"):  # (older builds loaded through FSTC_LIB for A/B runs lack these)
            lib.fst_compose_ex.argtypes = [vp, vp, C.c_uint32, vp, C.POINTER(vp)]
            lib.fst_compose_batch_ex.argtypes = [C.c_int32, C.POINTER(vp), C.POINTER(vp), C.c_uint32, vp,
                                                 C.POINTER(vp)]
            lib.fst_copy_provenance_to_host.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, vp]
            lib.fst_grad_scatter.argtypes = [vp, vp, vp, C.c_int64, vp, C.c_int64, vp]
        if hasattr(lib, "fst_compose_chain"):
            lib.fst_copy_pair_f_to_host.argtypes = [vp, vp, vp]
            lib.fst_compose_chain.argtypes = [C.c_int32, C.POINTER(vp), C.c_uint32, vp, C.POINTER(vp)]
        if hasattr(lib, "fst_forward_score"):
            lib.fst_forward_score.argtypes = [vp, vp, C.POINTER(C.c_double), vp]
        lib.fst_level_sizes.argtypes = [vp, C.c_int32, vp, C.c_int32]
        lib.fst_level_sizes.restype = C.c_int32
        lib.fst_adjacency.argtypes = [vp, C.c_int32, C.c_int32, vp, vp]
        lib.fst_set_profiling.argtypes = [C.c_int32]
        lib.fst_set_profiling.restype = None
        lib.fst_set_tile_mode.argtypes = [C.c_int32]
        lib.fst_set_tile_mode.restype = None
        lib.fst_set_wave_mode.argtypes = [C.c_int32]
        lib.fst_set_wave_mode.restype = None
        lib.fst_launch_count.restype = C.c_int64
        lib.fst_last_error.restype = C.c_char_p
        lib.fst_version.restype = C.c_char_p
        lib.fst_comm_unique_id.argtypes = [vp]
        lib.fst_comm_init.argtypes = [C.c_int32, C.c_int32, vp, C.POINTER(vp)]
        lib.fst_comm_destroy.argtypes = [vp]
        lib.fst_comm_destroy.restype = None
        lib.fst_compose_sharded.argtypes = [vp, vp, vp, vp, C.POINTER(vp)]
        lib.fst_compose_sharded_local.argtypes = [vp, vp, C.c_int32, vp, C.POINTER(vp)]
        lib.fst_shard_info.argtypes = [vp, C.POINTER(fst_shard_desc)]
        for name in ("fst_create", "fst_compose", "fst_compose_batch", "fst_info", "fst_copy_to_host",
                     "fst_get_stats", "fst_adjacency", "fst_comm_unique_id", "fst_comm_init",
                     "fst_compose_sharded", "fst_compose_sharded_local", "fst_shard_info", "fst_copy_arcs_to_host"):
            getattr(lib, name).restype = C.c_int
        _lib = lib
        return lib


def _check(st: int):
    if st != 0:
        raise FstError(st, load_library().fst_last_error().decode())


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


# ------------------------------------------------------------------------------------------ ABI
def fst_create(fst_like, stream=None) -> "Fst":
    """fst_like: an object with num_states, row_ptr, ilabel, olabel, dst, weight, is_start,
    is_accept as numpy arrays (host upload) or torch CUDA tensors (device)."""
    lib = load_library()
    arrays = [fst_like.row_ptr, fst_like.ilabel, fst_like.olabel, fst_like.dst, fst_like.weight,
              fst_like.is_start, fst_like.is_accept]
    dtypes = [np.int64, np.int32, np.int32, np.int32, np.float32, np.uint8, np.uint8]
    keep = []
    if all(hasattr(a, "data_ptr") for a in arrays):  # torch tensors
        import torch
        ptrs = []
        for a, dt in zip(arrays, dtypes):
            assert a.is_cuda and a.is_contiguous() and a.element_size() == np.dtype(dt).itemsize
            ptrs.append(a.data_ptr() if a.numel() else None)
        mem = FST_MEM_DEVICE
        E = int(arrays[1].numel())
    else:
        ptrs = []
        for a, dt in zip(arrays, dtypes):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            ptrs.append(a.ctypes.data if a.size else None)
        mem = FST_MEM_HOST
        E = int(keep[1].size)
    d = fst_desc(int(fst_like.num_states), E, *ptrs, mem)
    h = C.c_void_p()
    _check(lib.fst_create(C.byref(d), _stream_ptr(stream), C.byref(h)))
    return Fst(h)


def _flags(provenance: bool, eps_filter: bool) -> int:
    return (FST_COMPOSE_PROVENANCE if provenance else 0) | (FST_COMPOSE_EPS_FILTER if eps_filter else 0)


def fst_compose(a: "Fst", b: "Fst", stream=None, provenance: bool = False, eps_filter: bool = False) -> "Fst":
    """C = trim(A o B); provenance=True also records each arc's (arc_a, arc_b); eps_filter=True runs
    the three-state eps-filtered variant (states (pair_a, pair_b, pair_f)) (fst_compose_ex)."""
    lib = load_library()
    h = C.c_void_p()
    if provenance or eps_filter:
        _check(lib.fst_compose_ex(a.handle, b.handle, _flags(provenance, eps_filter), _stream_ptr(stream),
                                  C.byref(h)))
    else:
        _check(lib.fst_compose(a.handle, b.handle, _stream_ptr(stream), C.byref(h)))
    return Fst(h)


def fst_compose_ex(a: "Fst", b: "Fst", flags: int, stream=None) -> "Fst":
    lib = load_library()
    h = C.c_void_p()
    _check(lib.fst_compose_ex(a.handle, b.handle, flags, _stream_ptr(stream), C.byref(h)))
    return Fst(h)


def fst_compose_batch(a: Sequence["Fst"], b: Sequence["Fst"], stream=None, provenance: bool = False,
                      eps_filter: bool = False) -> List["Fst"]:
    lib = load_library()
    n = len(a)
    assert len(b) == n
    A = (C.c_void_p * n)(*[x.handle for x in a])
    B = (C.c_void_p * n)(*[x.handle for x in b])
    out = (C.c_void_p * n)()
    if provenance or eps_filter:
        _check(lib.fst_compose_batch_ex(n, A, B, _flags(provenance, eps_filter), _stream_ptr(stream), out))
    else:
        _check(lib.fst_compose_batch(n, A, B, _stream_ptr(stream), out))
    return [Fst(C.c_void_p(out[i])) for i in range(n)]


def fst_compose_chain(graphs: Sequence["Fst"], stream=None, eps_filter: bool = False) -> "Fst":
    """N-way composition: ((g0 o g1) o g2) o ... (left fold on the GPU, intermediates freed)."""
    lib = load_library()
    n = len(graphs)
    G = (C.c_void_p * n)(*[x.handle for x in graphs])
    h = C.c_void_p()
    _check(lib.fst_compose_chain(n, G, _flags(False, eps_filter), _stream_ptr(stream), C.byref(h)))
    return Fst(h)


def fst_forward_score(h: "Fst", alpha=None, stream=None) -> float:
    """Log-semiring forward score of an acyclic graph (float64); alpha: optional CUDA float64 tensor
    [num_states] receiving alpha."""
    lib = load_library()
    if alpha is not None and (not alpha.is_cuda or str(alpha.dtype) != "torch.float64" or not alpha.is_contiguous()
                              or alpha.numel() < h.num_states):
        raise FstError(1, "fst_forward_score: alpha must be a contiguous CUDA float64 tensor [num_states]")
    tot = C.c_double()
    _check(lib.fst_forward_score(h.handle, _stream_ptr(stream), C.byref(tot),
                                 alpha.data_ptr() if alpha is not None and alpha.numel() else None))
    return float(tot.value)


def fst_grad_scatter(c: "Fst", grad_c, grad_a=None, grad_b=None, stream=None):
    """Accumulates dL/dw_c (CUDA float32 tensor [E_C]) into grad_a [E_A] / grad_b [E_B] (CUDA float32
    tensors, +=) through the provenance of c (composed with provenance=True)."""
    lib = load_library()
    for t in (grad_c, grad_a, grad_b):
        if t is not None and (not t.is_cuda or str(t.dtype) != "torch.float32" or not t.is_contiguous()):
            raise FstError(1, "fst_grad_scatter: gradients must be contiguous CUDA float32 tensors")
    ptr = lambda t: t.data_ptr() if t is not None and t.numel() else None
    _check(lib.fst_grad_scatter(c.handle, ptr(grad_c), ptr(grad_a), 0 if grad_a is None else grad_a.numel(),
                                ptr(grad_b), 0 if grad_b is None else grad_b.numel(), _stream_ptr(stream)))


def fst_compose_sharded_local(a: "Fst", b: "Fst", world: int, stream=None) -> List["Fst"]:
    """All `world` shards of the sharded composition in this process (one device)."""
    lib = load_library()
    out = (C.c_void_p * world)()
    _check(lib.fst_compose_sharded_local(a.handle, b.handle, world, _stream_ptr(stream), out))
    return [Fst(C.c_void_p(out[i])) for i in range(world)]


class Comm:
    """NCCL communicator of the sharded mode (one rank per GPU).  Bootstrap: rank 0 calls
    ``Comm.unique_id()``, the caller broadcasts the 128 bytes (e.g. torch.distributed), then every
    rank builds ``Comm(world, rank, uid)``."""

    def __init__(self, world: int, rank: int, uid: bytes):
        lib = load_library()
        buf = C.create_string_buffer(bytes(uid), 128)
        self.handle = C.c_void_p()
        _check(lib.fst_comm_init(world, rank, buf, C.byref(self.handle)))
        self.world, self.rank = world, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(load_library().fst_comm_unique_id(buf))
        return buf.raw

    def close(self):
        if self.handle and self.handle.value:
            load_library().fst_comm_destroy(self.handle)
        self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fst_compose_sharded(a: "Fst", b: "Fst", comm: Comm, stream=None) -> "Fst":
    lib = load_library()
    h = C.c_void_p()
    _check(lib.fst_compose_sharded(a.handle, b.handle, comm.handle, _stream_ptr(stream), C.byref(h)))
    return Fst(h)


def fst_set_profiling(on: bool):
    load_library().fst_set_profiling(1 if on else 0)


def fst_set_tile_mode(mode: int):
    """0 = never use the tile kernels, 1 = automatic (default), 2 = whenever the inputs fit."""
    load_library().fst_set_tile_mode(int(mode))


def fst_set_wave_mode(mode: int):
    """Wave path (row-by-row stages for topologically numbered A): 0 = never, 1 = automatic (default),
    2 = whenever the inputs qualify."""
    load_library().fst_set_wave_mode(int(mode))


def fst_launch_count() -> int:
    return int(load_library().fst_launch_count())


def fst_version() -> str:
    return load_library().fst_version().decode()


class _DeviceArray:
    """__cuda_array_interface__ over library-owned device memory; holds its Fst alive."""

    def __init__(self, owner: "Fst", ptr: int, n: int, typestr: str):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr if n else 0, False),
                                         "version": 3, "strides": None}


class Fst:
    """Owning wrapper of an fst_handle (freed on garbage collection or ``free()``)."""

    def __init__(self, handle: C.c_void_p):
        self.handle = handle

    def free(self):
        if self.handle and self.handle.value:
            load_library().fst_free(self.handle)
        self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def info(self) -> fst_view:
        v = fst_view()
        _check(load_library().fst_info(self.handle, C.byref(v)))
        return v

    @property
    def num_states(self) -> int:
        return int(self.info().num_states)

    @property
    def num_arcs(self) -> int:
        return int(self.info().num_arcs)

    def to_host(self, stream=None) -> Dict[str, np.ndarray]:
        """fst_copy_to_host into fresh numpy arrays (pair_a/pair_b for composed graphs)."""
        v = self.info()
        V, E = int(v.num_states), int(v.num_arcs)
        out = {"num_states": V, "num_arcs": E,
               "row_ptr": np.zeros(V + 1, np.int64), "ilabel": np.zeros(E, np.int32),
               "olabel": np.zeros(E, np.int32), "dst": np.zeros(E, np.int32), "weight": np.zeros(E, np.float32),
               "is_start": np.zeros(V, np.uint8), "is_accept": np.zeros(V, np.uint8)}
        composed = bool(v.pair_a)
        if composed:
            out["pair_a"] = np.zeros(V, np.int32)
            out["pair_b"] = np.zeros(V, np.int32)
        ptr = lambda k: out[k].ctypes.data if k in out and out[k].size else None
        _check(load_library().fst_copy_to_host(self.handle, _stream_ptr(stream), ptr("row_ptr"), ptr("ilabel"),
                                               ptr("olabel"), ptr("dst"), ptr("weight"), ptr("is_start"),
                                               ptr("is_accept"), ptr("pair_a"), ptr("pair_b")))
        if v.arc_a:
            out["arc_a"], out["arc_b"] = self.provenance(stream)
        if v.pair_f:
            out["pair_f"] = self.pair_f(stream)
        return out

    def pair_f(self, stream=None) -> np.ndarray:
        """eps-filter state of every state (handles composed with eps_filter=True)."""
        V = self.num_states
        out = np.zeros(V, np.int32)
        _check(load_library().fst_copy_pair_f_to_host(self.handle, _stream_ptr(stream), out.ctypes.data if V else None))
        return out

    def device_tensors(self) -> Dict[str, "object"]:
        """Zero-copy torch CUDA tensors over the handle's device arrays (fst_info pointers).  Each tensor
        keeps this handle alive (the library owns the memory until every view and the handle are gone);
        treat them as read-only.  Keys: row_ptr, ilabel, olabel, dst, weight, is_start, is_accept, and
        pair_a / pair_b / pair_f / arc_a / arc_b when present."""
        import torch
        v = self.info()
        V, E = int(v.num_states), int(v.num_arcs)
        spec = [("row_ptr", v.row_ptr, V + 1, "<i8"), ("ilabel", v.ilabel, E, "<i4"), ("olabel", v.olabel, E, "<i4"),
                ("dst", v.dst, E, "<i4"), ("weight", v.weight, E, "<f4"), ("is_start", v.is_start, V, "|u1"),
                ("is_accept", v.is_accept, V, "|u1"), ("pair_a", v.pair_a, V, "<i4"), ("pair_b", v.pair_b, V, "<i4"),
                ("pair_f", v.pair_f, V, "<i4"), ("arc_a", v.arc_a, E, "<i4"), ("arc_b", v.arc_b, E, "<i4")]
        out = {}
        for name, ptr, n, typestr in spec:
            if not ptr and n > 0:
                continue
            out[name] = torch.as_tensor(_DeviceArray(self, ptr or 0, n, typestr), device="cuda")
        return out

    def provenance(self, stream=None):
        """(arc_a, arc_b) int32 arrays [E] (handles composed with provenance=True)."""
        E = self.num_arcs
        aa, ab = np.zeros(E, np.int32), np.zeros(E, np.int32)
        _check(load_library().fst_copy_provenance_to_host(self.handle, _stream_ptr(stream), 0, E,
                                                          aa.ctypes.data if E else None,
                                                          ab.ctypes.data if E else None))
        return aa, ab

    def state_arrays(self, stream=None) -> Dict[str, np.ndarray]:
        """Per-state arrays only (row_ptr, flags, pair_a/pair_b) -- no arcs."""
        v = self.info()
        V = int(v.num_states)
        out = {"num_states": V, "num_arcs": int(v.num_arcs), "row_ptr": np.zeros(V + 1, np.int64),
               "is_start": np.zeros(V, np.uint8), "is_accept": np.zeros(V, np.uint8),
               "pair_a": np.zeros(V, np.int32), "pair_b": np.zeros(V, np.int32)}
        ptr = lambda k: out[k].ctypes.data if out[k].size else None
        _check(load_library().fst_copy_to_host(self.handle, _stream_ptr(stream), ptr("row_ptr"), None, None, None,
                                               None, ptr("is_start"), ptr("is_accept"),
                                               ptr("pair_a") if v.pair_a else None, ptr("pair_b") if v.pair_b else None))
        return out

    def arcs_range(self, first: int, count: int, stream=None) -> Dict[str, np.ndarray]:
        out = {"ilabel": np.zeros(count, np.int32), "olabel": np.zeros(count, np.int32),
               "dst": np.zeros(count, np.int32), "weight": np.zeros(count, np.float32)}
        p = [out[k].ctypes.data if count else None for k in ("ilabel", "olabel", "dst", "weight")]
        _check(load_library().fst_copy_arcs_to_host(self.handle, _stream_ptr(stream), first, count, *p))
        return out

    def stats(self) -> dict:
        s = fst_compose_stats()
        _check(load_library().fst_get_stats(self.handle, C.byref(s)))
        return s.as_dict()

    def shard_info(self) -> dict:
        d = fst_shard_desc()
        _check(load_library().fst_shard_info(self.handle, C.byref(d)))
        return d.as_dict()

    def level_sizes(self, stage: int) -> List[int]:
        lib = load_library()
        n = lib.fst_level_sizes(self.handle, stage, None, 0)
        if n < 0:
            raise FstError(1, "not a composed handle")
        buf = np.zeros(max(n, 1), np.int64)
        lib.fst_level_sizes(self.handle, stage, buf.ctypes.data, n)
        return [int(x) for x in buf[:n]]

    def adjacency(self, role: int, match_on_olabel: bool):
        v = self.info()
        off = np.zeros(int(v.num_states) + 1, np.int64)
        arcs = np.zeros(max(1, int(v.num_arcs)), np.int64)
        _check(load_library().fst_adjacency(self.handle, role, 1 if match_on_olabel else 0, off.ctypes.data,
                                            arcs.ctypes.data))
        return off, arcs[: int(v.num_arcs)]


def compose(A, B, stream=None, provenance: bool = False, eps_filter: bool = False) -> Dict[str, np.ndarray]:
    """Convenience: host arrays in, composed graph (numpy, GPU numbering) out."""
    a = fst_create(A, stream)
    b = fst_create(B, stream)
    c = fst_compose(a, b, stream, provenance=provenance, eps_filter=eps_filter)
    return c.to_host(stream)
