"""Thin Python binding of libmsort.so (include/msort.h): argument marshalling only.

Every step of the sort runs in the library's sm_100a CUDA kernels; PyTorch
supplies device memory (workspace from its caching allocator), the current
stream and process groups.  There is no CPU fallback: if the library is not
built, importing this package raises.

Names follow the C ABI (msort_sort, msort_sort_pairs, msort_sort_distributed,
...).  `sort`, `sort_pairs` are functional conveniences that work on a clone
(the paper's sorts are pure functions).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSORT_LIB") or os.path.join(_PKG, "lib", "libmsort.so")

MSORT_INT32, MSORT_UINT32, MSORT_INT64, MSORT_UINT64, MSORT_NONE = 0, 1, 2, 3, 255
MSORT_PROFILE_CLASSES = 8
PROFILE_CLASS_NAMES = ("tile_sort", "partition", "merge_pass", "splitter", "kway_merge", "nccl",
                       "exchange", "key_range")

_TORCH_DT = {torch.int32: MSORT_INT32, torch.int64: MSORT_INT64}
if hasattr(torch, "uint32"):
    _TORCH_DT[torch.uint32] = MSORT_UINT32
if hasattr(torch, "uint64"):
    _TORCH_DT[torch.uint64] = MSORT_UINT64
_NP_DT = {np.dtype(np.int32): MSORT_INT32, np.dtype(np.uint32): MSORT_UINT32,
          np.dtype(np.int64): MSORT_INT64, np.dtype(np.uint64): MSORT_UINT64}

EXPORTED = (
    "msort_sort", "msort_sort_pairs", "msort_workspace_bytes", "msort_sort_ws",
    "msort_sort_out_ws", "msort_sort_distributed_out_ws",
    "msort_comm_unique_id", "msort_comm_init", "msort_comm_destroy", "msort_sort_distributed",
    "msort_sort_distributed_ws", "msort_sort_distributed_emulated", "msort_plan_rounds",
    "msort_plan_candidates_per_round", "msort_plan_init", "msort_plan_candidates",
    "msort_plan_narrow", "msort_plan_fill", "msort_status_string", "msort_last_error",
    "msort_profile_enable", "msort_profile_reset", "msort_profile_read", "msort_launch_count",
    "msort_tile_size", "msort_debug_set_quad", "msort_sort_host", "msort_debug_set_exchange",
    "msort_segmented_workspace_bytes", "msort_sort_segmented",
    "msort_sort_distributed_tree", "msort_sort_distributed_tree_emulated",
    "msort_plan_tree_rounds", "msort_plan_tree_role", "msort_comm_wrap",
    "msort_merge_runs", "msort_merge_runs_workspace_bytes", "msort_debug_tile_sort",
    "msort_comm_reserve", "msort_sort_distributed_host", "msort_comm_set_exchange",
)


class MsortError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_2211_16479_b200/build.py` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    c = ctypes
    vp, sz, i32, i64p = c.c_void_p, c.c_size_t, c.c_int, c.POINTER(c.c_int64)
    u64p = c.POINTER(c.c_uint64)
    L.msort_sort.argtypes = [vp, sz, i32, vp]
    L.msort_sort_pairs.argtypes = [vp, vp, sz, i32, i32, vp]
    L.msort_workspace_bytes.argtypes = [sz, i32, i32, i32, c.POINTER(c.c_size_t)]
    L.msort_sort_ws.argtypes = [vp, vp, sz, i32, i32, vp, sz, vp]
    L.msort_sort_out_ws.argtypes = [vp, vp, vp, vp, sz, i32, i32, vp, sz, vp]
    L.msort_sort_host.argtypes = [vp, vp, vp, vp, sz, i32, i32, vp, vp, vp, sz, vp]
    L.msort_sort_distributed_out_ws.argtypes = [vp, vp, vp, vp, sz, i32, i32, vp, vp, sz, vp,
                                                i64p]
    L.msort_comm_unique_id.argtypes = [vp]
    L.msort_comm_init.argtypes = [vp, i32, i32, c.POINTER(vp)]
    L.msort_comm_destroy.argtypes = [vp]
    L.msort_comm_wrap.argtypes = [vp, c.POINTER(vp)]
    L.msort_comm_reserve.argtypes = [vp, sz, i32, i32, vp]
    L.msort_comm_set_exchange.argtypes = [vp, i32]
    L.msort_sort_distributed_host.argtypes = [vp, vp, vp, vp, sz, i32, i32, vp, vp, vp, vp, sz, vp]
    L.msort_sort_distributed.argtypes = [vp, vp, sz, i32, i32, vp, vp, i64p]
    L.msort_sort_distributed_ws.argtypes = [vp, vp, sz, i32, i32, vp, vp, sz, vp, i64p]
    L.msort_sort_distributed_emulated.argtypes = [c.POINTER(vp), c.POINTER(vp),
                                                  c.POINTER(c.c_size_t), i32, i32, i32,
                                                  c.POINTER(vp), sz, vp, i64p]
    L.msort_plan_rounds.argtypes = [i32]
    L.msort_plan_rounds.restype = i32
    L.msort_plan_candidates_per_round.restype = i32
    L.msort_plan_init.argtypes = [i32, i32, u64p]
    L.msort_plan_candidates.argtypes = [i32, u64p, u64p]
    L.msort_plan_narrow.argtypes = [i32, u64p, u64p, u64p]
    L.msort_plan_fill.argtypes = [i32, u64p, u64p, i64p]
    L.msort_status_string.argtypes = [i32]
    L.msort_status_string.restype = c.c_char_p
    L.msort_last_error.restype = c.c_char_p
    L.msort_profile_enable.argtypes = [i32]
    L.msort_profile_read.argtypes = [i64p, c.POINTER(c.c_double)]
    L.msort_launch_count.restype = c.c_int64
    L.msort_segmented_workspace_bytes.argtypes = [c.c_size_t, c.c_size_t, i32, i32,
                                                  c.POINTER(c.c_size_t)]
    L.msort_sort_segmented.argtypes = [c.c_void_p, c.c_void_p, c.c_size_t, i64p, c.c_size_t, i32,
                                       i32, c.c_void_p, c.c_size_t, c.c_void_p]
    L.msort_sort_distributed_tree.argtypes = [vp, vp, sz, i32, i32, vp, vp, vp, sz, vp, i64p]
    L.msort_sort_distributed_tree_emulated.argtypes = [c.POINTER(vp), c.POINTER(vp),
                                                       c.POINTER(c.c_size_t), i32, i32, i32, vp,
                                                       vp, vp]
    L.msort_plan_tree_rounds.argtypes = [i32]
    L.msort_plan_tree_rounds.restype = i32
    L.msort_plan_tree_role.argtypes = [i32, i32, i32, c.POINTER(i32)]
    L.msort_plan_tree_role.restype = i32
    L.msort_merge_runs_workspace_bytes.argtypes = [sz, i32, i32, i32, c.POINTER(c.c_size_t)]
    L.msort_merge_runs.argtypes = [vp, vp, i64p, i32, vp, vp, i32, i32, vp, sz, vp]
    L.msort_debug_tile_sort.argtypes = [vp, vp, c.c_int64, i32, vp]
    L.msort_debug_tile_sort.restype = i32
    L.msort_tile_size.argtypes = [i32, i32]
    L.msort_tile_size.restype = i32
    for f in ("msort_sort", "msort_sort_pairs", "msort_workspace_bytes", "msort_sort_ws",
              "msort_sort_out_ws", "msort_sort_distributed_out_ws", "msort_sort_host",
              "msort_comm_unique_id", "msort_comm_init", "msort_comm_destroy",
              "msort_sort_distributed", "msort_sort_distributed_ws",
              "msort_sort_distributed_emulated", "msort_plan_init", "msort_plan_candidates",
              "msort_plan_narrow", "msort_plan_fill", "msort_profile_read",
              "msort_segmented_workspace_bytes", "msort_sort_segmented",
              "msort_sort_distributed_tree", "msort_sort_distributed_tree_emulated",
              "msort_comm_wrap", "msort_merge_runs", "msort_merge_runs_workspace_bytes",
              "msort_comm_reserve", "msort_sort_distributed_host"):
        getattr(L, f).restype = i32
    return L


lib = _load()


def _check(st: int, what: str):
    if st != 0:
        name = lib.msort_status_string(st).decode()
        detail = lib.msort_last_error().decode()
        raise MsortError(f"{what}: {name}: {detail}")


def _dt(t: torch.Tensor) -> int:
    try:
        return _TORCH_DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported key dtype {t.dtype}") from None


def _vdt(v: torch.Tensor | None) -> int:
    if v is None:
        return MSORT_NONE
    if v.dtype == torch.int32:
        return MSORT_INT32
    if hasattr(torch, "uint32") and v.dtype == torch.uint32:
        return MSORT_UINT32
    raise TypeError(f"payload must be a 4-byte integer tensor, got {v.dtype}")


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _keep_for(ws: torch.Tensor, stream) -> None:
    """A workspace allocated here on the current stream but used on another
    one: keep the caching allocator from reusing it before that stream is
    done with it."""
    if stream is not None and isinstance(stream, torch.cuda.Stream):
        ws.record_stream(stream)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_NULL = _Null()


def _on(device):
    """torch.cuda.device(device), skipped when it is already current (the
    context manager costs microseconds per call; small sorts notice)."""
    if device.index is None or device.index == torch.cuda.current_device():
        return _NULL
    return torch.cuda.device(device)


def _check_tensor(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous() or t.dim() != 1:
        raise ValueError(f"{name} must be a contiguous 1-D tensor")


def msort_workspace_bytes(n: int, key_dtype: int, val_dtype: int = MSORT_NONE,
                          world: int = 1) -> int:
    out = ctypes.c_size_t()
    _check(lib.msort_workspace_bytes(n, key_dtype, val_dtype, world, ctypes.byref(out)),
           "msort_workspace_bytes")
    return out.value


def workspace(n: int, keys_dtype: torch.dtype, with_vals: bool, world: int = 1,
              device=None) -> torch.Tensor:
    """A workspace tensor from PyTorch's caching allocator."""
    nb = msort_workspace_bytes(n, _TORCH_DT[keys_dtype], MSORT_UINT32 if with_vals else MSORT_NONE,
                               world)
    return torch.empty(max(nb, 1), dtype=torch.uint8, device=device)


def msort_sort(keys: torch.Tensor, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Stable ascending sort of a 1-D CUDA tensor in place."""
    return msort_sort_pairs(keys, None, ws=ws, stream=stream)[0]


def msort_sort_pairs(keys: torch.Tensor, vals: torch.Tensor | None, ws: torch.Tensor | None = None,
                     stream=None):
    """Stable sort of (keys, vals) by key, in place; ties keep input order."""
    _check_tensor(keys, "keys")
    if vals is not None:
        _check_tensor(vals, "vals")
        if vals.numel() != keys.numel() or vals.device != keys.device:
            raise ValueError("keys/vals size or device mismatch")
    n = keys.numel()
    kd, vd = _dt(keys), _vdt(vals)
    if n < 2:
        return keys, vals
    if ws is None:
        ws = workspace(n, keys.dtype, vals is not None, device=keys.device)
        _keep_for(ws, stream)
    with _on(keys.device):
        _check(lib.msort_sort_ws(_ptr(keys), _ptr(vals), n, kd, vd, _ptr(ws), ws.numel(),
                                 ctypes.c_void_p(_stream(stream))), "msort_sort_ws")
    return keys, vals


def msort_sort_out(in_keys: torch.Tensor, keys_out: torch.Tensor, in_vals=None, vals_out=None,
                   ws: torch.Tensor | None = None, stream=None):
    """Out-of-place stable sort: in_keys (unchanged) -> keys_out."""
    _check_tensor(in_keys, "in_keys")
    _check_tensor(keys_out, "keys_out")
    if keys_out.numel() != in_keys.numel() or keys_out.dtype != in_keys.dtype:
        raise ValueError("in/out keys mismatch")
    if (in_vals is None) != (vals_out is None):
        raise ValueError("give both in_vals and vals_out, or neither")
    n = in_keys.numel()
    kd, vd = _dt(in_keys), _vdt(in_vals)
    if ws is None:
        ws = workspace(n, in_keys.dtype, in_vals is not None, device=in_keys.device)
        _keep_for(ws, stream)
    with _on(in_keys.device):
        _check(lib.msort_sort_out_ws(_ptr(in_keys), _ptr(in_vals), _ptr(keys_out), _ptr(vals_out),
                                     n, kd, vd, _ptr(ws), ws.numel(),
                                     ctypes.c_void_p(_stream(stream))), "msort_sort_out_ws")
    return keys_out, vals_out


def msort_sort_host(host_keys: torch.Tensor, host_keys_out: torch.Tensor, dev_keys: torch.Tensor,
                    host_vals=None, host_vals_out=None, dev_vals=None,
                    ws: torch.Tensor | None = None, stream=None):
    """End-to-end sort of host tensors (include/msort.h msort_sort_host):
    upload into dev_keys (dev_vals), sort there, copy back to host_keys_out
    (host_vals_out); asynchronous on `stream` for pinned host tensors."""
    for t, name in ((host_keys, "host_keys"), (host_keys_out, "host_keys_out")):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous host tensor")
    _check_tensor(dev_keys, "dev_keys")
    n = host_keys.numel()
    if host_keys_out.numel() != n or dev_keys.numel() != n:
        raise ValueError("host/device sizes differ")
    kd, vd = _dt(dev_keys), _vdt(dev_vals)
    if ws is None:
        ws = workspace(n, dev_keys.dtype, dev_vals is not None, device=dev_keys.device)
        _keep_for(ws, stream)
    with _on(dev_keys.device):
        _check(lib.msort_sort_host(_ptr(host_keys), _ptr(host_vals), _ptr(host_keys_out),
                                   _ptr(host_vals_out), n, kd, vd, _ptr(dev_keys), _ptr(dev_vals),
                                   _ptr(ws), ws.numel(), ctypes.c_void_p(_stream(stream))),
               "msort_sort_host")
    return host_keys_out, host_vals_out


def msort_segmented_workspace_bytes(n: int, nseg: int, key_dtype: int,
                                    val_dtype: int = MSORT_NONE) -> int:
    out = ctypes.c_size_t()
    _check(lib.msort_segmented_workspace_bytes(n, nseg, key_dtype, val_dtype, ctypes.byref(out)),
           "msort_segmented_workspace_bytes")
    return out.value


def msort_sort_segmented(keys: torch.Tensor, seg_offsets, vals: torch.Tensor | None = None,
                         ws: torch.Tensor | None = None, stream=None):
    """Batched stable sort of every segment keys[off[i]:off[i+1]] (and vals)
    in place (include/msort.h msort_sort_segmented).  seg_offsets: nseg + 1
    int64 offsets -- a CUDA int64 tensor (used in place: classified on the
    device, one stream synchronisation), or a list / numpy array / CPU tensor
    (read on the host, fully asynchronous)."""
    _check_tensor(keys, "keys")
    if vals is not None:
        _check_tensor(vals, "vals")
        if vals.numel() != keys.numel() or vals.device != keys.device:
            raise ValueError("keys/vals size or device mismatch")
    dev_off = isinstance(seg_offsets, torch.Tensor) and seg_offsets.is_cuda
    if dev_off:
        off_t = seg_offsets.to(torch.int64).contiguous()
        if off_t.dim() != 1 or off_t.numel() < 1 or off_t.device != keys.device:
            raise ValueError("seg_offsets must be 1-D with nseg + 1 offsets on the keys' device")
        off_ptr = ctypes.cast(ctypes.c_void_p(off_t.data_ptr()), ctypes.POINTER(ctypes.c_int64))
        nseg = off_t.numel() - 1
    else:
        if isinstance(seg_offsets, torch.Tensor):
            seg_offsets = seg_offsets.detach().numpy()
        off = np.ascontiguousarray(np.asarray(seg_offsets, dtype=np.int64))
        if off.ndim != 1 or off.size < 1:
            raise ValueError("seg_offsets must be a 1-D array of nseg + 1 offsets")
        off_ptr = off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        nseg = off.size - 1
    n = keys.numel()
    kd, vd = _dt(keys), _vdt(vals)
    if ws is None:
        nb = msort_segmented_workspace_bytes(n, nseg, kd, vd)
        ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=keys.device)
        _keep_for(ws, stream)
    with _on(keys.device):
        _check(lib.msort_sort_segmented(_ptr(keys), _ptr(vals), n, off_ptr, nseg,
                                        kd, vd, _ptr(ws), ws.numel(),
                                        ctypes.c_void_p(_stream(stream))), "msort_sort_segmented")
    return keys, vals


def msort_merge_runs(in_keys: torch.Tensor, run_offsets, keys_out: torch.Tensor | None = None,
                     in_vals: torch.Tensor | None = None, vals_out: torch.Tensor | None = None,
                     ws: torch.Tensor | None = None, stream=None):
    """Stable merge of p sorted runs in_keys[off[j]:off[j+1]] (include/msort.h
    msort_merge_runs; ties to the lower run).  run_offsets: p + 1 host
    offsets (list / numpy / CPU tensor).  Returns (keys_out, vals_out)."""
    _check_tensor(in_keys, "in_keys")
    if isinstance(run_offsets, torch.Tensor):
        run_offsets = run_offsets.detach().cpu().numpy()
    off = np.ascontiguousarray(np.asarray(run_offsets, dtype=np.int64))
    if off.ndim != 1 or off.size < 2:
        raise ValueError("run_offsets must hold p + 1 >= 2 offsets")
    p = off.size - 1
    n = in_keys.numel()
    if int(off[-1]) != n:
        raise ValueError("run_offsets[-1] must equal in_keys.numel()")
    if keys_out is None:
        keys_out = torch.empty_like(in_keys)
    _check_tensor(keys_out, "keys_out")
    if keys_out.numel() != n or keys_out.dtype != in_keys.dtype or keys_out.device != in_keys.device:
        raise ValueError("keys_out must match in_keys (size, dtype, device)")
    if in_vals is not None:
        _check_tensor(in_vals, "in_vals")
        if in_vals.numel() != n or in_vals.device != in_keys.device:
            raise ValueError("in_vals must match in_keys (size, device)")
        if vals_out is None:
            vals_out = torch.empty_like(in_vals)
        _check_tensor(vals_out, "vals_out")
        if vals_out.numel() != n or vals_out.dtype != in_vals.dtype:
            raise ValueError("vals_out must match in_vals")
    kd, vd = _dt(in_keys), _vdt(in_vals)
    if ws is None:
        nb = ctypes.c_size_t()
        _check(lib.msort_merge_runs_workspace_bytes(n, p, kd, vd, ctypes.byref(nb)),
               "msort_merge_runs_workspace_bytes")
        ws = torch.empty(max(nb.value, 256), dtype=torch.uint8, device=in_keys.device)
        _keep_for(ws, stream)
    with _on(in_keys.device):
        _check(lib.msort_merge_runs(_ptr(in_keys), _ptr(in_vals),
                                    off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), p,
                                    _ptr(keys_out), _ptr(vals_out), kd, vd, _ptr(ws), ws.numel(),
                                    ctypes.c_void_p(_stream(stream))), "msort_merge_runs")
    return keys_out, vals_out


def sort(x: torch.Tensor) -> torch.Tensor:
    """Functional stable sort: returns a sorted copy (input unchanged)."""
    return msort_sort_out(x, torch.empty_like(x))[0]


def sort_(x: torch.Tensor) -> torch.Tensor:
    """In-place stable sort on the current stream (SURVEY §8(b) Python layer)."""
    return msort_sort(x)


def sort_pairs(k: torch.Tensor, v: torch.Tensor):
    """Functional stable sort of (k, v) by key: sorted copies (inputs unchanged)."""
    return msort_sort_pairs(k.clone(), v.clone())


# (group, device index) -> Comm.  Keyed by the group OBJECT (hashed by
# identity and kept alive by the key), so a destroyed group whose id() is
# reused can never pick up a stale communicator.
_COMMS = {}


def sort_distributed(x: torch.Tensor, group=None, vals: torch.Tensor | None = None):
    """In-place collective stable sort over a torch NCCL process group (default:
    the world): rank r ends with the global positions [K_r, K_r + n_r) of the
    rank-major concatenation.  The library's own NCCL communicator for the
    group is created on first use (id broadcast over the group) and cached."""
    import torch.distributed as dist

    g = group if group is not None else dist.group.WORLD
    key = (g, x.device.index)
    comm = _COMMS.get(key)
    if comm is None:
        comm = _COMMS[key] = Comm(group)
    msort_sort_distributed(x, comm, vals=vals)
    return (x, vals) if vals is not None else x


# ------------------------------------------------------------- distributed
class Comm:
    """An NCCL communicator of libmsort built over a torch process group
    (the unique id is broadcast over the group)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        idb = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(lib.msort_comm_unique_id(idb), "msort_comm_unique_id")
        obj = [bytes(idb.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        idb = ctypes.create_string_buffer(obj[0], 128)
        h = ctypes.c_void_p()
        _check(lib.msort_comm_init(idb, self.rank, self.world, ctypes.byref(h)), "msort_comm_init")
        self.handle = h

    def reserve(self, n_max: int, keys_dtype=torch.int32, with_vals: bool = False, stream=None):
        """Collective: reserve the pull exchange for up to n_max local keys
        (include/msort.h msort_comm_reserve); afterwards pull-mode sorts of
        keys with 3..8 ranks run without host synchronisation."""
        _check(lib.msort_comm_reserve(self.handle, int(n_max), _TORCH_DT[keys_dtype],
                                      MSORT_UINT32 if with_vals else MSORT_NONE,
                                      ctypes.c_void_p(_stream(stream))), "msort_comm_reserve")

    def set_exchange(self, mode: int) -> None:
        """Exchange mode of this communicator's distributed calls
        (include/msort.h msort_comm_set_exchange): 0 NCCL all-to-all + k-way
        merge, 1 fused pull exchange, -1 the process default.  Every rank
        must set the same mode."""
        _check(lib.msort_comm_set_exchange(self.handle, int(mode)), "msort_comm_set_exchange")

    def close(self):
        if self.handle:
            _check(lib.msort_comm_destroy(self.handle), "msort_comm_destroy")
            self.handle = None

    @classmethod
    def from_torch(cls, group=None, device=None):
        """Wrap the NCCL communicator of a torch NCCL process group
        (include/msort.h msort_comm_wrap; non-owning).  One collective is run
        first so torch has created its communicator."""
        import torch.distributed as dist

        dev = device or torch.device("cuda", torch.cuda.current_device())
        pg = group or dist.group.WORLD
        t = torch.zeros(1, device=dev)
        dist.all_reduce(t, group=pg)
        torch.cuda.synchronize(dev)
        ptr = pg._get_backend(dev)._comm_ptr()
        self = cls.__new__(cls)
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        h = ctypes.c_void_p()
        _check(lib.msort_comm_wrap(ctypes.c_void_p(ptr), ctypes.byref(h)), "msort_comm_wrap")
        self.handle = h
        return self


def msort_sort_distributed(keys: torch.Tensor, comm: Comm, vals: torch.Tensor | None = None,
                           ws: torch.Tensor | None = None, stream=None,
                           return_split: bool = False):
    """Collective stable sort: rank r ends with global positions [K_r, K_r+n_r)."""
    _check_tensor(keys, "keys")
    if vals is not None:
        _check_tensor(vals, "vals")
        if vals.numel() != keys.numel() or vals.device != keys.device:
            raise ValueError("keys/vals size or device mismatch")
    n = keys.numel()
    kd, vd = _dt(keys), _vdt(vals)
    if ws is None:
        ws = workspace(n, keys.dtype, vals is not None, world=comm.world, device=keys.device)
    # the split matrix only when asked for: fetching it is a host synchronisation
    split = np.zeros((comm.world + 1) * comm.world, dtype=np.int64) if return_split else None
    sp = split.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if return_split else None
    with _on(keys.device):
        _check(lib.msort_sort_distributed_ws(
            _ptr(keys), _ptr(vals), n, kd, vd, comm.handle, _ptr(ws), ws.numel(),
            ctypes.c_void_p(_stream(stream)), sp), "msort_sort_distributed_ws")
    if return_split:
        return keys, vals, split.reshape(comm.world + 1, comm.world)
    return keys, vals


def msort_sort_distributed_host(host_keys: torch.Tensor, host_keys_out: torch.Tensor,
                                dev_keys: torch.Tensor, comm: Comm, host_vals=None,
                                host_vals_out=None, dev_vals=None, ws: torch.Tensor | None = None,
                                stream=None):
    """End-to-end collective sort of host tensors (include/msort.h
    msort_sort_distributed_host): upload into dev_keys, sort across the
    ranks, copy this rank's slice back to host_keys_out."""
    for t, name in ((host_keys, "host_keys"), (host_keys_out, "host_keys_out")):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous host tensor")
    _check_tensor(dev_keys, "dev_keys")
    n = host_keys.numel()
    if host_keys_out.numel() != n or dev_keys.numel() != n:
        raise ValueError("host/device sizes differ")
    kd, vd = _dt(dev_keys), _vdt(dev_vals)
    if ws is None:
        ws = workspace(n, dev_keys.dtype, dev_vals is not None, world=comm.world,
                       device=dev_keys.device)
    with _on(dev_keys.device):
        _check(lib.msort_sort_distributed_host(
            _ptr(host_keys), _ptr(host_vals), _ptr(host_keys_out), _ptr(host_vals_out), n, kd, vd,
            comm.handle, _ptr(dev_keys), _ptr(dev_vals), _ptr(ws), ws.numel(),
            ctypes.c_void_p(_stream(stream))), "msort_sort_distributed_host")
    return host_keys_out, host_vals_out


def msort_sort_distributed_out(in_keys: torch.Tensor, keys_out: torch.Tensor, comm: Comm,
                               in_vals=None, vals_out=None, ws: torch.Tensor | None = None,
                               stream=None, return_split: bool = False):
    """Out-of-place collective sort: in_keys (unchanged) -> this rank's slice."""
    _check_tensor(in_keys, "in_keys")
    _check_tensor(keys_out, "keys_out")
    if keys_out.numel() != in_keys.numel() or keys_out.dtype != in_keys.dtype or \
            keys_out.device != in_keys.device:
        raise ValueError("in/out keys mismatch (size, dtype or device)")
    if (in_vals is None) != (vals_out is None):
        raise ValueError("give both in_vals and vals_out, or neither")
    if in_vals is not None:
        _check_tensor(in_vals, "in_vals")
        _check_tensor(vals_out, "vals_out")
        if in_vals.numel() != in_keys.numel() or vals_out.numel() != in_keys.numel() or \
                in_vals.dtype != vals_out.dtype:
            raise ValueError("in_vals / vals_out must match the keys' size and each other's dtype")
    n = in_keys.numel()
    kd, vd = _dt(in_keys), _vdt(in_vals)
    if ws is None:
        ws = workspace(n, in_keys.dtype, in_vals is not None, world=comm.world,
                       device=in_keys.device)
    split = np.zeros((comm.world + 1) * comm.world, dtype=np.int64) if return_split else None
    sp = split.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if return_split else None
    with _on(in_keys.device):
        _check(lib.msort_sort_distributed_out_ws(
            _ptr(in_keys), _ptr(in_vals), _ptr(keys_out), _ptr(vals_out), n, kd, vd, comm.handle,
            _ptr(ws), ws.numel(), ctypes.c_void_p(_stream(stream)), sp),
            "msort_sort_distributed_out_ws")
    if return_split:
        return keys_out, vals_out, split.reshape(comm.world + 1, comm.world)
    return keys_out, vals_out


def msort_sort_distributed_emulated(keys: list, vals: list | None = None, stream=None):
    """p virtual ranks on one GPU (same kernels/planning; collectives emulated
    on the device).  Sorts every shard tensor in place; returns the split matrix."""
    p = len(keys)
    for k in keys:
        _check_tensor(k, "keys")
    kd = _dt(keys[0])
    vd = _vdt(vals[0]) if vals else MSORT_NONE
    nmax = max(k.numel() for k in keys)
    wsb = msort_workspace_bytes(nmax, kd, vd, p)
    wss = [torch.empty(wsb, dtype=torch.uint8, device=keys[0].device) for _ in range(p)]
    VP = ctypes.c_void_p * p
    kp = VP(*[k.data_ptr() for k in keys])
    vp = VP(*[v.data_ptr() for v in vals]) if vals else None
    np_ = (ctypes.c_size_t * p)(*[k.numel() for k in keys])
    wp = VP(*[w.data_ptr() for w in wss])
    split = np.zeros((p + 1) * p, dtype=np.int64)
    with _on(keys[0].device):
        _check(lib.msort_sort_distributed_emulated(
            kp, vp, np_, p, kd, vd, wp, wsb, ctypes.c_void_p(_stream(stream)),
            split.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
            "msort_sort_distributed_emulated")
    return split.reshape(p + 1, p)


def msort_sort_distributed_tree(in_keys: torch.Tensor, comm: Comm, in_vals=None,
                                root_keys: torch.Tensor | None = None, root_vals=None,
                                stream=None):
    """The paper's rank-tree gather (include/msort.h msort_sort_distributed_tree):
    collective; rank 0 receives every rank's keys, sorted, in root_keys (allocated
    here with the global size when None).  Returns (root_keys, root_vals) on rank 0,
    (None, None) elsewhere.  Ties come out in the tree's rank order."""
    import torch.distributed as dist

    _check_tensor(in_keys, "in_keys")
    n = in_keys.numel()
    kd, vd = _dt(in_keys), _vdt(in_vals)
    t = torch.tensor([n], dtype=torch.int64, device=in_keys.device)
    dist.all_reduce(t, group=getattr(comm, "group", None))  # the global size, over comm's group
    total = int(t.item())
    if comm.rank == 0 and root_keys is None:
        root_keys = torch.empty(total, dtype=in_keys.dtype, device=in_keys.device)
        if in_vals is not None:
            root_vals = torch.empty(total, dtype=in_vals.dtype, device=in_keys.device)
    cap = root_keys.numel() if root_keys is not None else 0
    tot = ctypes.c_int64()
    with _on(in_keys.device):
        _check(lib.msort_sort_distributed_tree(
            _ptr(in_keys), _ptr(in_vals), n, kd, vd, comm.handle, _ptr(root_keys),
            _ptr(root_vals), cap, ctypes.c_void_p(_stream(stream)), ctypes.byref(tot)),
            "msort_sort_distributed_tree")
    return (root_keys, root_vals) if comm.rank == 0 else (None, None)


def msort_sort_distributed_tree_emulated(keys: list, vals: list | None = None, stream=None):
    """The rank-tree gather for p virtual ranks on one GPU: returns the root's
    (keys, vals) -- every shard's elements, sorted, ties in the tree's rank order."""
    p = len(keys)
    for k in keys:
        _check_tensor(k, "keys")
    kd = _dt(keys[0])
    vd = _vdt(vals[0]) if vals else MSORT_NONE
    total = sum(k.numel() for k in keys)
    rk = torch.empty(total, dtype=keys[0].dtype, device=keys[0].device)
    rv = torch.empty(total, dtype=vals[0].dtype, device=keys[0].device) if vals else None
    VP = ctypes.c_void_p * p
    kp = VP(*[k.data_ptr() for k in keys])
    vp = VP(*[v.data_ptr() for v in vals]) if vals else None
    np_ = (ctypes.c_size_t * p)(*[k.numel() for k in keys])
    with _on(keys[0].device):
        _check(lib.msort_sort_distributed_tree_emulated(
            kp, vp, np_, p, kd, vd, _ptr(rk), _ptr(rv), ctypes.c_void_p(_stream(stream))),
            "msort_sort_distributed_tree_emulated")
    return rk, rv


# --------------------------------------------------- planning (host side)
def _u64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def plan_rounds(key_dtype: int) -> int:
    return lib.msort_plan_rounds(key_dtype)


def plan_candidates_per_round() -> int:
    return lib.msort_plan_candidates_per_round()


def plan_init(key_dtype: int, world: int) -> np.ndarray:
    lohi = np.zeros(2 * max(world - 1, 0) + 1, dtype=np.uint64)
    _check(lib.msort_plan_init(key_dtype, world, _u64p(lohi)), "msort_plan_init")
    return lohi[: 2 * (world - 1)]


def plan_candidates(world: int, lohi: np.ndarray) -> np.ndarray:
    B = plan_candidates_per_round()
    lohi = np.ascontiguousarray(lohi, dtype=np.uint64)
    cand = np.zeros(max(world - 1, 0) * B + 1, dtype=np.uint64)
    _check(lib.msort_plan_candidates(world, _u64p(lohi), _u64p(cand)), "msort_plan_candidates")
    return cand[: (world - 1) * B].reshape(world - 1, B)


def plan_narrow(world: int, K: np.ndarray, total: np.ndarray, lohi: np.ndarray) -> np.ndarray:
    K = np.ascontiguousarray(K, dtype=np.uint64)
    total = np.ascontiguousarray(total, dtype=np.uint64).ravel()
    lohi = np.ascontiguousarray(lohi, dtype=np.uint64).copy()
    _check(lib.msort_plan_narrow(world, _u64p(K), _u64p(total), _u64p(lohi)), "msort_plan_narrow")
    return lohi


def plan_fill(world: int, K: np.ndarray, lteq: np.ndarray) -> np.ndarray:
    K = np.ascontiguousarray(K, dtype=np.uint64)
    lteq = np.ascontiguousarray(lteq, dtype=np.uint64).ravel()
    if lteq.size == 0:
        lteq = np.zeros(1, dtype=np.uint64)
    out = np.zeros((world + 1) * world, dtype=np.int64)
    _check(lib.msort_plan_fill(world, _u64p(K), _u64p(lteq),
                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
           "msort_plan_fill")
    return out.reshape(world + 1, world)


def plan_tree(world: int, rank: int):
    """[(role, peer)] per round of the rank tree (include/msort.h
    msort_plan_tree_role): role 0 idle, 1 parent (receive from peer), 2 child
    (send to peer)."""
    out = []
    for t in range(lib.msort_plan_tree_rounds(world)):
        peer = ctypes.c_int(-1)
        role = lib.msort_plan_tree_role(world, rank, t, ctypes.byref(peer))
        out.append((role, peer.value))
    return out


# --------------------------------------------------------------- profiling
def profile_enable(on: bool = True):
    lib.msort_profile_enable(1 if on else 0)


def profile_reset():
    lib.msort_profile_reset()


def profile_read():
    la = (ctypes.c_int64 * MSORT_PROFILE_CLASSES)()
    ms = (ctypes.c_double * MSORT_PROFILE_CLASSES)()
    _check(lib.msort_profile_read(la, ms), "msort_profile_read")
    return {PROFILE_CLASS_NAMES[i]: (int(la[i]), float(ms[i])) for i in range(MSORT_PROFILE_CLASSES)}


def launch_count() -> int:
    return int(lib.msort_launch_count())


def set_exchange_mode(mode: int) -> None:
    """Distributed exchange (include/msort.h msort_debug_set_exchange): 0 NCCL
    all-to-all then k-way merge, 1 pull (first merge round reads the peers'
    sorted segments in place)."""
    lib.msort_debug_set_exchange(int(mode))


def set_quad_mode(mode: int) -> None:
    """Merge-level grouping for keys-only sorts (include/msort.h
    msort_debug_set_quad): 0 two-way levels only (default), 5 K6 4-way passes."""
    lib.msort_debug_set_quad(int(mode))


def tile_size(key_dtype: int, val_dtype: int = MSORT_NONE) -> int:
    return int(lib.msort_tile_size(key_dtype, val_dtype))
