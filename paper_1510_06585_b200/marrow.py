"""Thin ctypes binding of libmarrow.so (include/marrow.h).

Function names are the C-ABI names; this module only marshals arguments and
turns error codes into ``MwError``.  Every step of the hot path runs inside
libmarrow's sm_100a kernels: there is no Python or CPU fallback, and importing
this module fails loudly if the library has not been built.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmarrow.so")

# ---------------------------------------------------------------- constants (marrow.h)
MW_OK = 0
(MW_E_INVALID_SPEC, MW_E_EPU_NU, MW_E_INFEASIBLE_PARTITION, MW_E_SHAPE_MISMATCH,
 MW_E_MISSING_ITERATION_COUNT, MW_E_NOT_CONVERGED, MW_E_CUDA, MW_E_NCCL, MW_E_STATE,
 MW_E_OOM, MW_E_UNSUPPORTED) = range(1, 12)
MW_MERGE_ADD, MW_MERGE_SUB, MW_MERGE_MUL, MW_MERGE_DIV, MW_MERGE_USER = range(5)
MW_REDUCE_SUM, MW_REDUCE_MAX, MW_REDUCE_MIN = range(3)
MW_TERM_ABS, MW_TERM_SQUARE = 0, 1
MW_SCALAR_SQRT, MW_SCALAR_SCALE = 0, 1
# host callbacks (NEXT-4): merging function and host-side loop condition
_MERGE_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_void_p)
_COND_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p)
(MW_VK_SAXPY, MW_VK_RGBA, MW_VK_U8, MW_VK_U8_2D, MW_VK_NBODY, MW_VK_VEC1, MW_VK_VEC2,
 MW_VK_TERMS, MW_VK_ACCEL, MW_VK_TRAITS, MW_VK_SCALAR, MW_VK_CPLX) = range(1, 13)
MW_DT_U8, MW_DT_F32, MW_DT_F64, MW_DT_I64 = 1, 2, 3, 4
MW_PARTITION, MW_COPY = 0, 1
MW_LOC_DEVICE, MW_LOC_HOST = 0, 1
MW_TRANSPORT_AUTO, MW_TRANSPORT_NCCL, MW_TRANSPORT_LOOPBACK = 0, 1, 2
MW_BALANCE_PROPORTIONAL, MW_BALANCE_ABS = 0, 1
MW_PROV_BUILT, MW_PROV_DERIVED, MW_PROV_BALANCED = 0, 1, 2
MW_KB_NONE, MW_KB_EXACT, MW_KB_SCT, MW_KB_WORKLOAD, MW_KB_DIMENSIONALITY = range(5)
(MW_TUNE_RGBA_TMA, MW_TUNE_RGBA_UNROLL, MW_TUNE_HYST_PLANES, MW_TUNE_HYST_T, MW_TUNE_HYST_ROWS,
 MW_TUNE_NBODY_SPLIT, MW_TUNE_U8_TMA, MW_TUNE_HYST_FUSED, MW_TUNE_GRAPH_LANES, MW_TUNE_FFT_4STEP,
 MW_TUNE_COUNT) = range(11)
(MW_KC_SAXPY, MW_KC_RGBA, MW_KC_U8, MW_KC_STENCIL, MW_KC_NBODY, MW_KC_REDUCE,
 MW_KC_TRAITS, MW_KC_FFT, MW_KC_COUNT) = range(9)


class MwError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        self.status = status
        super().__init__(f"{fn}: {_name(status)}: {msg}")


class mw_alloc_fns(ctypes.Structure):
    _fields_ = [("alloc", ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                           ctypes.c_void_p)),
                ("free", ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)),
                ("user", ctypes.c_void_p)]


class mw_arg(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("ndim", ctypes.c_int32),
                ("shape", ctypes.c_int64 * 4), ("mode", ctypes.c_int32),
                ("location", ctypes.c_int32), ("local_offset", ctypes.c_int64),
                ("local_rows", ctypes.c_int64)]


class mw_balance_params(ctypes.Structure):
    _fields_ = [("weight", ctypes.c_double), ("max_dev", ctypes.c_double),
                ("c_factor", ctypes.c_double), ("trigger", ctypes.c_double),
                ("mode", ctypes.c_int32)]


class mw_balance_state(ctypes.Structure):
    _fields_ = [("lbt", ctypes.c_double), ("active", ctypes.c_int32),
                ("abs_last_dir", ctypes.c_int32), ("abs_t", ctypes.c_double),
                ("abs_count", ctypes.c_int32), ("pad", ctypes.c_int32), ("runs", ctypes.c_int64)]


class mw_profile_params(ctypes.Structure):
    _fields_ = [("executions", ctypes.c_int32), ("precision_ms", ctypes.c_double),
                ("max_dist_iters", ctypes.c_int32)]


class mw_managed_params(ctypes.Structure):
    _fields_ = [("balance", mw_balance_params), ("build_profiles", ctypes.c_int32),
                ("profile", mw_profile_params)]


(MW_MANAGED_NO_KNOWLEDGE, MW_MANAGED_FROM_KB, MW_MANAGED_DERIVED, MW_MANAGED_RECURRENT,
 MW_MANAGED_ADJUSTED, MW_MANAGED_BUILT) = range(6)
MANAGED_ACTIONS = ("no_knowledge", "from_kb", "derived", "recurrent", "adjusted", "built")

_lib = None
_P = ctypes.POINTER
_vp, _i32, _i64, _f32, _f64, _u32 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_float, ctypes.c_double, ctypes.c_uint32)
_node_pp = _P(_vp)

# name -> argtypes (restype mw_status unless listed in _RES)
_SIG = {
    "mw_status_string": [_i32],
    "mw_last_error": [_vp],
    "mw_abi_version": [],
    "mw_nccl_unique_id": [_P(ctypes.c_uint8)],
    "mw_ctx_create": [_i32, _i32, _i32, _i32, _P(ctypes.c_uint8), _i32, _P(mw_alloc_fns), _P(_vp)],
    "mw_ctx_destroy": [_vp],
    "mw_ctx_info": [_vp, _P(_i32), _P(_i32), _P(_i32), _P(_i32), _P(_i32)],
    "mw_kernel_saxpy": [_f32, _node_pp],
    "mw_kernel_gauss_noise": [_u32, _i32, _node_pp],
    "mw_kernel_solarize": [_i32, _node_pp],
    "mw_kernel_mirror": [_node_pp],
    "mw_kernel_segment": [_i32, _i32, _node_pp],
    "mw_kernel_hysteresis_step": [_node_pp],
    "mw_kernel_hysteresis_finalize": [_node_pp],
    "mw_kernel_nbody_step": [_f32, _f32, _node_pp],
    "mw_kernel_nbody_accel": [_f32, _node_pp],
    "mw_kernel_map_identity": [_node_pp],
    "mw_kernel_map_product": [_node_pp],
    "mw_kernel_debug_traits": [_i64, _i64, _i32, _node_pp],
    "mw_kernel_fft": [_i32, _i32, _node_pp],
    "mw_pipeline": [_P(_vp), _i32, _node_pp],
    "mw_map": [_vp, _node_pp],
    "mw_map_reduce": [_vp, _i32, _node_pp],
    "mw_kernel_reduce": [_i32, _node_pp],
    "mw_kernel_term_map": [_i32, _node_pp],
    "mw_kernel_scalar_map": [_i32, _f64, _node_pp],
    "mw_map_reduce_sct": [_vp, _vp, _node_pp],
    "mw_ctx_set_monitoring": [_vp, _i32],
    "mw_ctx_set_staging_overlap": [_vp, _i32],
    "mw_ctx_set_run_pipelining": [_vp, _i32],
    "mw_map_reduce_user": [_vp, _MERGE_FN, _vp, _node_pp],
    "mw_loop_host": [_vp, _i64, _COND_FN, _vp, _node_pp],
    "mw_loop_for": [_vp, _i64, _node_pp],
    "mw_loop_while_changed": [_vp, _i64, _i32, _node_pp],
    "mw_node_retain": [_vp],
    "mw_node_release": [_vp],
    "mw_node_id": [_vp, _P(ctypes.c_uint8)],
    "mw_node_signature": [_vp, _P(_i32), _P(_i32)],
    "mw_kernel_execution_order": [_vp, _P(_i64), _i32, _P(_i32), _P(_i64)],
    "mw_granule": [_vp, _P(_i64)],
    "mw_partition_plan": [_i64, _i64, _P(_f64), _i32, _i32, _P(_i64), _P(_i64)],
    "mw_set_distribution": [_vp, _P(_f64), _i32],
    "mw_get_distribution": [_vp, _P(_f64), _i32],
    "mw_partition": [_vp, _vp, _i64, _P(_i64), _P(_i64)],
    "mw_run": [_vp, _vp, _P(mw_arg), _i32, _vp, _P(_vp)],
    "mw_future_wait": [_vp],
    "mw_future_query": [_vp, _P(_i32)],
    "mw_future_result": [_vp, _P(_f64), _i32],
    "mw_future_release": [_vp],
    "mw_last_timings": [_vp, _P(_f32), _i32, _P(_f32)],
    "mw_last_lengths": [_vp, _P(_i64), _i32],
    "mw_balance_defaults": [_P(mw_balance_params)],
    "mw_balance_step": [_P(mw_balance_params), _P(mw_balance_state), _P(_f32), _P(_i64),
                        _P(_f64), _i32, _P(_f64), _P(_i32)],
    "mw_rebalance": [_vp, _P(mw_balance_params), _P(_i32)],
    "mw_get_balance_state": [_vp, _P(mw_balance_state)],
    "mw_ctx_set_slowdown": [_vp, _i32, _f32],
    "mw_stats_enable": [_vp, _i32],
    "mw_graph_capture": [_vp, _vp, _P(mw_arg), _i32, _vp, _P(_vp)],
    "mw_graph_capture_many": [_vp, _vp, _P(mw_arg), _i32, _i32, _vp, _P(_vp)],
    "mw_graph_launch": [_vp, _vp],
    "mw_graph_result": [_vp, _P(_f64), _i32],
    "mw_graph_kernels": [_vp, _P(_i64)],
    "mw_graph_destroy": [_vp],
    "mw_kernel_stats": [_vp, _i32, _P(_f64), _P(_i64)],
    "mw_ctx_launch_count": [_vp, _P(_i64)],
    "mw_ctx_set_tuning": [_vp, _i32, _i32],
    "mw_kb_open": [ctypes.c_char_p, _P(_vp)],
    "mw_kb_save": [_vp],
    "mw_kb_close": [_vp],
    "mw_kb_count": [_vp, _P(_i32)],
    "mw_kb_store": [_vp, _vp, _P(_i64), _i32, _P(_i32), _P(_f64), _i32, _f64, _i32],
    "mw_kb_lookup": [_vp, _vp, _P(_i64), _i32, _P(_i32), _P(_f64), _i32, _P(_i32)],
    "mw_autotune": [_vp, _vp, _P(mw_arg), _i32, _vp, _i32, _vp, _P(_i32), _P(_f64)],
    "mw_ctx_get_tuning": [_vp, _i32, _P(_i32)],
    "mw_kb_find": [_vp, _vp, _P(_i64), _i32, _P(_i32), _P(_i32), _P(_f64)],
    "mw_ctx_set_device_class": [_vp, _i32, _i32, _f64],
    "mw_profile_defaults": [_P(mw_profile_params)],
    "mw_profile_build": [_vp, _vp, _P(mw_arg), _i32, _vp, _P(mw_profile_params), _vp, _P(_i32), _P(_f64),
                         _i32, _P(_f64), _P(_i32)],
    "mw_managed_defaults": [_P(mw_managed_params)],
    "mw_run_managed": [_vp, _vp, _P(mw_managed_params), _vp, _P(mw_arg), _i32, _vp, _P(_vp), _P(_i32)],
    "mw_managed_flush": [_vp],
}
_RES = {"mw_status_string": ctypes.c_char_p, "mw_last_error": ctypes.c_char_p,
        "mw_abi_version": _i32, "mw_node_retain": None, "mw_node_release": None,
        "mw_future_release": None, "mw_balance_defaults": None, "mw_profile_defaults": None,
        "mw_managed_defaults": None}
EXPORTS = tuple(_SIG)


def lib():
    """Load libmarrow.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run `python __graft_entry__.py` "
                              "(build) — the hot path has no non-CUDA implementation")
        L = ctypes.CDLL(_LIB_PATH)
        for name, argt in _SIG.items():
            fn = getattr(L, name)
            fn.argtypes = argt
            fn.restype = _RES.get(name, _i32)
        _lib = L
    return _lib


def _name(st):
    try:
        return lib().mw_status_string(st).decode()
    except Exception:  # pragma: no cover
        return str(st)


def _chk(st, fn):
    if st != MW_OK:
        raise MwError(st, fn, lib().mw_last_error(None).decode())


def _call(name, *args):
    _chk(getattr(lib(), name)(*args), name)


# ---------------------------------------------------------------- nodes
class Node:
    """Owning handle of an mw_node (released on garbage collection)."""

    def __init__(self, ptr, kids=()):
        self.ptr = ptr
        self._kids = kids

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.mw_node_release(self.ptr)
            self.ptr = None

    @property
    def _as_parameter_(self):
        return self.ptr


def _new(name, *args, kids=()):
    out = _vp()
    _call(name, *args, ctypes.byref(out))
    return Node(out, kids)


def mw_kernel_saxpy(a):
    return _new("mw_kernel_saxpy", _f32(a))


def mw_kernel_gauss_noise(seed, scale):
    return _new("mw_kernel_gauss_noise", _u32(seed & 0xFFFFFFFF), scale)


def mw_kernel_solarize(threshold):
    return _new("mw_kernel_solarize", threshold)


def mw_kernel_mirror():
    return _new("mw_kernel_mirror")


def mw_kernel_segment(lo, hi):
    return _new("mw_kernel_segment", lo, hi)


def mw_kernel_hysteresis_step():
    return _new("mw_kernel_hysteresis_step")


def mw_kernel_hysteresis_finalize():
    return _new("mw_kernel_hysteresis_finalize")


def mw_kernel_nbody_step(dt, eps2):
    return _new("mw_kernel_nbody_step", _f32(dt), _f32(eps2))


def mw_kernel_nbody_accel(eps2):
    return _new("mw_kernel_nbody_accel", _f32(eps2))


def mw_kernel_map_identity():
    return _new("mw_kernel_map_identity")


def mw_kernel_map_product():
    return _new("mw_kernel_map_product")


def mw_kernel_debug_traits(epu=1, nu=1, strict=False):
    return _new("mw_kernel_debug_traits", epu, nu, int(bool(strict)))


def mw_kernel_fft(log2n=16, inverse=False):
    """FFT of every row of a complex64 batch f32[B][2^log2n][2] (NEXT-3,
    P:729-732); inverse includes 1/N."""
    return _new("mw_kernel_fft", log2n, int(bool(inverse)))


def mw_pipeline(stages):
    arr = (_vp * len(stages))(*[s.ptr for s in stages])
    return _new("mw_pipeline", arr, len(stages), kids=tuple(stages))


def mw_map(tree):
    return _new("mw_map", tree.ptr, kids=(tree,))


def mw_map_reduce(map_stage, merge_op=MW_MERGE_ADD):
    return _new("mw_map_reduce", map_stage.ptr, merge_op, kids=(map_stage,))


def mw_kernel_reduce(op=MW_REDUCE_SUM):
    """Device reduction-stage leaf (NEXT-4, P:191 map_reduce(SCT, SCT))."""
    return _new("mw_kernel_reduce", op)


def mw_kernel_term_map(kind):
    """Reduction-stage term map (MW_TERM_ABS / MW_TERM_SQUARE), NEXT-4."""
    return _new("mw_kernel_term_map", kind)


def mw_kernel_scalar_map(kind, c=0.0):
    """Reduction-stage map of the reduced value (MW_SCALAR_SQRT / SCALE by c)."""
    return _new("mw_kernel_scalar_map", kind, _f64(c))


def mw_map_reduce_sct(map_stage, reduction_stage):
    """MapReduce whose reduction stage is a device SCT (mw_kernel_reduce)."""
    return _new("mw_map_reduce_sct", map_stage.ptr, reduction_stage.ptr,
                kids=(map_stage, reduction_stage))


def mw_loop_for(body, n):
    return _new("mw_loop_for", body.ptr, n, kids=(body,))


def mw_loop_while_changed(body, max_iters, check_every=1):
    return _new("mw_loop_while_changed", body.ptr, max_iters, check_every, kids=(body,))


def mw_map_reduce_user(map_stage, fn):
    """MapReduce with a user-defined merging function fn(acc, partial) -> float
    over the per-partition partial results (NEXT-4)."""
    cb = _MERGE_FN(lambda acc, part, _u: float(fn(acc, part)))
    return _new("mw_map_reduce_user", map_stage.ptr, cb, None, kids=(map_stage, cb))


def mw_loop_host(body, max_iters, cond):
    """Loop whose condition cond(iteration) -> bool runs on the host before
    every iteration (P:374-378 stages 1 and 3; NEXT-4)."""
    cb = _COND_FN(lambda it, _u: 1 if cond(it) else 0)
    return _new("mw_loop_host", body.ptr, max_iters, cb, None, kids=(body, cb))


def mw_node_id(node) -> bytes:
    buf = (ctypes.c_uint8 * 32)()
    _call("mw_node_id", node.ptr, buf)
    return bytes(buf)


def mw_node_signature(node):
    i, o = _i32(), _i32()
    _call("mw_node_signature", node.ptr, ctypes.byref(i), ctypes.byref(o))
    return i.value, o.value


def mw_kernel_execution_order(node, while_counts=()):
    wc = (_i64 * max(1, len(while_counts)))(*while_counts)
    n = _i64(0)
    st = lib().mw_kernel_execution_order(node.ptr, wc, len(while_counts), None, ctypes.byref(n))
    if st not in (MW_OK, MW_E_INVALID_SPEC) or (st == MW_E_INVALID_SPEC and n.value == 0):
        _chk(st, "mw_kernel_execution_order")
    out = (_i32 * max(1, n.value))()
    _call("mw_kernel_execution_order", node.ptr, wc, len(while_counts), out, ctypes.byref(n))
    return list(out[:n.value])


def mw_granule(node) -> int:
    g = _i64()
    _call("mw_granule", node.ptr, ctypes.byref(g))
    return g.value


def mw_partition_plan(L, g, fractions, strict=False):
    k = len(fractions)
    d = (_f64 * max(1, k))(*fractions)
    off, ln = (_i64 * max(1, k))(), (_i64 * max(1, k))()
    _call("mw_partition_plan", L, g, d, k, int(bool(strict)), off, ln)
    return list(off[:k]), list(ln[:k])


# ---------------------------------------------------------------- balance (pure host)
def mw_balance_defaults(mode=MW_BALANCE_PROPORTIONAL):
    p = mw_balance_params()
    lib().mw_balance_defaults(ctypes.byref(p))
    p.mode = mode
    return p


def mw_balance_step(params, state, per_part_ms, per_part_len, cur):
    n = len(cur)
    ms = (_f32 * n)(*per_part_ms)
    ln = (_i64 * n)(*per_part_len)
    cd = (_f64 * n)(*cur)
    nx = (_f64 * n)()
    trig = _i32()
    _call("mw_balance_step", ctypes.byref(params), ctypes.byref(state), ms, ln, cd, n, nx,
          ctypes.byref(trig))
    return list(nx), bool(trig.value)


# ---------------------------------------------------------------- context
def mw_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _call("mw_nccl_unique_id", buf)
    return bytes(buf)


class TorchAllocator:
    """mw_alloc_fns backed by PyTorch's caching allocator (PyTorch owns memory)."""

    def __init__(self, device):
        import torch
        self._torch = torch
        self.device = torch.device(device)
        self.live = {}

        @ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
        def _alloc(nbytes, stream, user):
            # the block belongs to the stream the library uses it on, so the
            # caching allocator never hands it to another stream while that
            # stream's kernels may still run (the library drains its streams
            # before it frees a buffer)
            try:
                if stream:
                    with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=self.device)):
                        t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
                else:
                    t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
                self.live[t.data_ptr()] = t
                return t.data_ptr()
            except Exception:
                return None

        @ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)
        def _free(ptr, user):
            self.live.pop(ptr, None)

        self._a, self._f = _alloc, _free
        self.fns = mw_alloc_fns(_alloc, _free, None)


class Ctx:
    def __init__(self, ptr, allocator):
        self.ptr = ptr
        self.allocator = allocator

    def __del__(self):
        self.destroy()

    def destroy(self):
        if getattr(self, "ptr", None) and _lib is not None:
            try:
                _reap_pending(all_of_ctx=self)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            _lib.mw_ctx_destroy(self.ptr)
            self.ptr = None

    @property
    def _as_parameter_(self):
        return self.ptr


def mw_ctx_create(device=0, rank=0, nranks=1, parts_per_rank=1, nccl_id=None, force_nccl=False,
                  torch_alloc=True, transport=None):
    """transport: MW_TRANSPORT_* (default AUTO, or NCCL when force_nccl)."""
    out = _vp()
    idbuf = (ctypes.c_uint8 * 128)(*nccl_id) if nccl_id is not None else None
    alloc = TorchAllocator(f"cuda:{device}") if torch_alloc else None
    if transport is None:
        transport = MW_TRANSPORT_NCCL if force_nccl else MW_TRANSPORT_AUTO
    _call("mw_ctx_create", device, rank, nranks, parts_per_rank, idbuf, int(transport),
          ctypes.byref(alloc.fns) if alloc else None, ctypes.byref(out))
    return Ctx(out, alloc)


def mw_ctx_destroy(ctx):
    ctx.destroy()


def mw_ctx_info(ctx):
    v = [_i32() for _ in range(5)]
    _call("mw_ctx_info", ctx.ptr, *[ctypes.byref(x) for x in v])
    return {"n_parts": v[0].value, "first_part": v[1].value, "parts_per_rank": v[2].value,
            "rank": v[3].value, "nranks": v[4].value}


def mw_set_distribution(ctx, fractions):
    d = (_f64 * len(fractions))(*fractions)
    _call("mw_set_distribution", ctx.ptr, d, len(fractions))


def mw_get_distribution(ctx):
    n = mw_ctx_info(ctx)["n_parts"]
    d = (_f64 * n)()
    _call("mw_get_distribution", ctx.ptr, d, n)
    return list(d)


def mw_partition(ctx, node, L):
    n = mw_ctx_info(ctx)["n_parts"]
    off, ln = (_i64 * n)(), (_i64 * n)()
    _call("mw_partition", ctx.ptr, node.ptr, L, off, ln)
    return list(off), list(ln)


# ---------------------------------------------------------------- args / run
_DT = {"uint8": MW_DT_U8, "float32": MW_DT_F32, "float64": MW_DT_F64, "int64": MW_DT_I64}


def arg(t, mode=MW_PARTITION, local_offset=0, global_shape=None):
    """mw_arg for a torch tensor (CUDA or host) or a numpy array (host).

    global_shape defaults to t.shape (the tensor holds the whole array);
    for a slice holding global rows [local_offset, local_offset + len(t)),
    pass the global shape."""
    a = mw_arg()
    if hasattr(t, "data_ptr"):
        ptr, shape, dt = t.data_ptr(), tuple(t.shape), str(t.dtype).replace("torch.", "")
        loc = MW_LOC_DEVICE if t.is_cuda else MW_LOC_HOST
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
    else:
        ptr, shape, dt = t.ctypes.data, tuple(t.shape), str(t.dtype)
        loc = MW_LOC_HOST
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
    gshape = tuple(global_shape) if global_shape is not None else shape
    a.ptr = ptr
    a.dtype = _DT[dt]
    a.ndim = len(gshape)
    for i, s in enumerate(gshape):
        a.shape[i] = s
    a.mode = mode
    a.location = loc
    a.local_offset = local_offset
    a.local_rows = shape[0] if len(shape) else 0
    a._owner = t   # keeps the buffer alive until the run's future is released
    return a


# Futures dropped while their run is still in flight: the handle and the
# argument owners are parked here (release order) and released once the run
# completes — checked oldest-first by every mw_run, so dropping a future never
# blocks and torch's caching allocator cannot hand a dropped argument's memory
# to a new tensor before the run has used it.
import collections as _collections
import threading as _threading

_pending = _collections.deque()
_pending_lock = _threading.RLock()   # ranks may be host threads (loopback transport)


_reaping = [False]


def _reap_pending(all_of_ctx=None):
    with _pending_lock:
        _reap_pending_locked(all_of_ctx)


def _reap_pending_locked(all_of_ctx):
    if _reaping[0]:   # re-entered from a destructor run by the garbage collector
        return
    _reaping[0] = True
    try:
        if all_of_ctx is not None:   # ctx teardown: release its parked futures
            for item in [it for it in _pending if it[1][2] is all_of_ctx]:
                _pending.remove(item)
                _lib.mw_future_release(item[0])
            return
        while _pending:
            item = _pending.popleft()
            d = _i32()
            if _lib.mw_future_query(item[0], ctypes.byref(d)) == MW_OK and not d.value:
                _pending.appendleft(item)   # oldest still in flight: stop
                break
            _lib.mw_future_release(item[0])
    finally:
        _reaping[0] = False


class Future:
    def __init__(self, ptr, keep):
        self.ptr = ptr
        self._keep = keep

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            if self._keep and getattr(self._keep[2], "ptr", None):
                with _pending_lock:
                    _pending.append((self.ptr, self._keep))   # maybe in flight: park it
            else:
                _lib.mw_future_release(self.ptr)
            self.ptr = None

    def wait(self):
        mw_future_wait(self)
        return self

    def result(self):
        return mw_future_result(self)


class ArgList:
    """The ctypes argument array of a run, built once: pass it to mw_run in
    place of a list to skip the per-call marshalling (repeated runs on the
    same buffers, e.g. a benchmark loop)."""
    __slots__ = ("arr", "n", "owners")

    def __init__(self, args):
        self.arr = (mw_arg * len(args))(*args)
        self.n = len(args)
        self.owners = [getattr(a, "_owner", None) for a in args]


_run_fn = None


def _current_stream_ptr():
    import torch
    try:
        return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())
    except AttributeError:  # pragma: no cover
        return torch.cuda.current_stream().cuda_stream


def mw_run(ctx, node, args, stream=None):
    """Enqueue a run on `stream` (torch.cuda.Stream or raw cudaStream_t int;
    default: torch's current stream).  args: a list of mw_arg or an ArgList."""
    global _run_fn
    if _run_fn is None:
        _run_fn = lib().mw_run
    if not isinstance(args, ArgList):
        args = ArgList(args)
    if stream is None:
        sp = _current_stream_ptr()
    else:
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    if len(_pending) > 32:   # amortised: one completion query per reclaimed run
        _reap_pending()
    out = _vp()
    st = _run_fn(ctx.ptr, node.ptr, args.arr, args.n, _vp(sp), ctypes.byref(out))
    if st != MW_OK:
        _chk(st, "mw_run")
    return Future(out, (args, node, ctx))


def mw_future_wait(f):
    _call("mw_future_wait", f.ptr)


def mw_future_query(f) -> bool:
    d = _i32()
    _call("mw_future_query", f.ptr, ctypes.byref(d))
    return bool(d.value)


def mw_future_result(f):
    """dict(reduced fp64, reduced32, executions, converged)."""
    out = (_f64 * 4)()
    _call("mw_future_result", f.ptr, out, 4)
    return {"reduced": out[0], "reduced32": out[1], "executions": int(out[2]),
            "converged": bool(out[3])}


def mw_future_release(f):
    if f.ptr:
        lib().mw_future_release(f.ptr)
        f.ptr = None


def mw_last_timings(ctx):
    n = mw_ctx_info(ctx)["n_parts"]
    ms, wall = (_f32 * n)(), _f32()
    _call("mw_last_timings", ctx.ptr, ms, n, ctypes.byref(wall))
    return list(ms), wall.value


def mw_last_lengths(ctx):
    n = mw_ctx_info(ctx)["n_parts"]
    ln = (_i64 * n)()
    _call("mw_last_lengths", ctx.ptr, ln, n)
    return list(ln)


def mw_rebalance(ctx, params=None) -> bool:
    p = params or mw_balance_defaults()
    t = _i32()
    _call("mw_rebalance", ctx.ptr, ctypes.byref(p), ctypes.byref(t))
    return bool(t.value)


def mw_get_balance_state(ctx):
    s = mw_balance_state()
    _call("mw_get_balance_state", ctx.ptr, ctypes.byref(s))
    return s


def mw_ctx_set_slowdown(ctx, part, factor):
    _call("mw_ctx_set_slowdown", ctx.ptr, part, _f32(factor))


def mw_ctx_launch_count(ctx) -> int:
    n = _i64()
    _call("mw_ctx_launch_count", ctx.ptr, ctypes.byref(n))
    return n.value


def mw_stats_enable(ctx, on=True):
    _call("mw_stats_enable", ctx.ptr, int(bool(on)))


def mw_kernel_stats(ctx, kernel_class):
    """(total event-measured ms, launches) of one kernel class since enabling."""
    ms, n = _f64(), _i64()
    _call("mw_kernel_stats", ctx.ptr, kernel_class, ctypes.byref(ms), ctypes.byref(n))
    return ms.value, n.value


class Graph:
    """Owning handle of an mw_graph (keeps its buffers and tree alive)."""

    def __init__(self, ptr, keep):
        self.ptr = ptr
        self._keep = keep

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.mw_graph_destroy(self.ptr)
            self.ptr = None

    def launch(self, stream=None):
        mw_graph_launch(self, stream)

    def result(self):
        out = (_f64 * 4)()
        _call("mw_graph_result", self.ptr, out, 4)
        return {"reduced": out[0], "reduced32": out[1], "executions": int(out[2]),
                "converged": bool(out[3])}

    @property
    def kernels(self):
        n = _i64()
        _call("mw_graph_kernels", self.ptr, ctypes.byref(n))
        return n.value


def _stream_arg(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return _vp(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def mw_graph_capture(ctx, node, args, stream=None):
    arr = (mw_arg * len(args))(*args)
    out = _vp()
    _call("mw_graph_capture", ctx.ptr, node.ptr, arr, len(args), _stream_arg(stream),
          ctypes.byref(out))
    return Graph(out, (arr, node, ctx, [getattr(a, "_owner", None) for a in args]))


def mw_graph_capture_many(ctx, node, arg_sets, stream=None):
    """One graph replaying len(arg_sets) back-to-back runs (set k on arg_sets[k])."""
    nargs = len(arg_sets[0])
    flat = [a for st in arg_sets for a in st]
    arr = (mw_arg * len(flat))(*flat)
    out = _vp()
    _call("mw_graph_capture_many", ctx.ptr, node.ptr, arr, nargs, len(arg_sets),
          _stream_arg(stream), ctypes.byref(out))
    return Graph(out, (arr, node, ctx, [getattr(a, "_owner", None) for a in flat]))


def mw_graph_launch(g, stream=None):
    _call("mw_graph_launch", g.ptr, _stream_arg(stream))


def mw_graph_destroy(g):
    if g.ptr:
        _call("mw_graph_destroy", g.ptr)
        g.ptr = None


def mw_ctx_set_monitoring(ctx, on=True):
    """Per-partition timing events on/off (on by default; needed by
    mw_last_timings / mw_rebalance)."""
    _call("mw_ctx_set_monitoring", ctx.ptr, int(bool(on)))


def mw_ctx_set_staging_overlap(ctx, on=True):
    """Host inputs are complete when mw_run is called: staged uploads overlap
    the previous run's downloads (no start barrier)."""
    _call("mw_ctx_set_staging_overlap", ctx.ptr, int(bool(on)))


def mw_ctx_set_run_pipelining(ctx, on=True):
    """Promise: no foreign work between this ctx's runs writes what they read;
    independent fused-chain runs then overlap their predecessor's drain."""
    _call("mw_ctx_set_run_pipelining", ctx.ptr, int(bool(on)))


def mw_ctx_set_tuning(ctx, knob, value):
    _call("mw_ctx_set_tuning", ctx.ptr, knob, value)


def mw_ctx_get_tuning(ctx, knob) -> int:
    v = _i32()
    _call("mw_ctx_get_tuning", ctx.ptr, knob, ctypes.byref(v))
    return v.value


class KB:
    """Owning handle of an mw_kb (saved and freed on close / garbage collection)."""

    def __init__(self, ptr):
        self.ptr = ptr

    def close(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _call("mw_kb_close", self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mw_kb_open(path=None):
    out = _vp()
    _call("mw_kb_open", (path or "").encode(), ctypes.byref(out))
    return KB(out)


def mw_kb_save(kb):
    _call("mw_kb_save", kb.ptr)


def mw_kb_close(kb):
    kb.close()


def mw_kb_count(kb) -> int:
    n = _i32()
    _call("mw_kb_count", kb.ptr, ctypes.byref(n))
    return n.value


def mw_kb_store(kb, node, dims, tune, fractions, best_ms, provenance=MW_PROV_BUILT):
    d = (_i64 * max(1, len(dims)))(*dims)
    tn = (_i32 * MW_TUNE_COUNT)(*tune)
    fr = (_f64 * max(1, len(fractions)))(*fractions)
    _call("mw_kb_store", kb.ptr, node.ptr, d, len(dims), tn, fr, len(fractions), best_ms, provenance)


def mw_kb_lookup(kb, node, dims, nparts=0):
    """-> (scope, tune list or None, fractions list or None)."""
    d = (_i64 * max(1, len(dims)))(*dims)
    tn = (_i32 * MW_TUNE_COUNT)()
    fr = (_f64 * max(1, nparts))()
    sc = _i32()
    _call("mw_kb_lookup", kb.ptr, node.ptr, d, len(dims), tn, fr if nparts else None, nparts,
          ctypes.byref(sc))
    if sc.value == MW_KB_NONE:
        return MW_KB_NONE, None, None
    return sc.value, list(tn), (list(fr)[:nparts] if nparts else None)


def mw_autotune(ctx, node, args, stream=None, reps=3, kb=None):
    """Profile building over the tuning knobs; returns (tune list, best ms per run)."""
    arr = (mw_arg * len(args))(*args)
    tn = (_i32 * MW_TUNE_COUNT)()
    ms = _f64()
    _call("mw_autotune", ctx.ptr, node.ptr, arr, len(args), _stream_arg(stream), reps,
          kb.ptr if kb is not None else None, tn, ctypes.byref(ms))
    return list(tn), ms.value


# ---------------------------------------------------------------- NEXT-2 / NEXT-4
def mw_kb_find(kb, node, dims):
    """-> (found, provenance, best_ms) of the exact (SCT, workload) record."""
    d = (_i64 * max(1, len(dims)))(*dims)
    f, p, ms = _i32(), _i32(), _f64()
    _call("mw_kb_find", kb.ptr, node.ptr, d, len(dims), ctypes.byref(f), ctypes.byref(p), ctypes.byref(ms))
    return bool(f.value), p.value, ms.value


def mw_ctx_set_device_class(ctx, part, cls, rel_perf=1.0):
    """Partition `part` runs on device class `cls` with relative performance
    rel_perf; the distribution becomes proportional to it."""
    _call("mw_ctx_set_device_class", ctx.ptr, part, cls, _f64(rel_perf))


def mw_profile_defaults():
    p = mw_profile_params()
    lib().mw_profile_defaults(ctypes.byref(p))
    return p


def mw_profile_build(ctx, node, args, params=None, kb=None, stream=None):
    """Alg. 1 profile building; -> dict(tune, fractions, best_ms, runs)."""
    arr = (mw_arg * len(args))(*args)
    n = mw_ctx_info(ctx)["n_parts"]
    tn, fr = (_i32 * MW_TUNE_COUNT)(), (_f64 * n)()
    ms, runs = _f64(), _i32()
    p = params or mw_profile_defaults()
    _call("mw_profile_build", ctx.ptr, node.ptr, arr, len(args), _stream_arg(stream), ctypes.byref(p),
          kb.ptr if kb is not None else None, tn, fr, n, ctypes.byref(ms), ctypes.byref(runs))
    return {"tune": list(tn), "fractions": list(fr), "best_ms": ms.value, "runs": runs.value}


def mw_managed_defaults():
    p = mw_managed_params()
    lib().mw_managed_defaults(ctypes.byref(p))
    return p


def mw_run_managed(ctx, kb, node, args, params=None, stream=None):
    """Fig. 5 decision process around a run; -> (Future, action name)."""
    al = args if isinstance(args, ArgList) else ArgList(args)
    out, act = _vp(), _i32()
    p = params or mw_managed_defaults()
    _call("mw_run_managed", ctx.ptr, kb.ptr, ctypes.byref(p), node.ptr, al.arr, al.n, _stream_arg(stream),
          ctypes.byref(out), ctypes.byref(act))
    return Future(out, (al, node, ctx)), MANAGED_ACTIONS[act.value]


def mw_managed_flush(ctx):
    _call("mw_managed_flush", ctx.ptr)
