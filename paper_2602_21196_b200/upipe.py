"""Thin ctypes binding of libupipe (include/upipe.h), same names as the C ABI.

Argument marshalling only: every step of the layer runs in the CUDA kernels of
``libupipe.so``. PyTorch supplies device memory, streams and (for the NCCL
transport) the process group used to broadcast the NCCL unique id. There is no
CPU or PyTorch fallback: if the library is missing, the import of any entry
point raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_uint8, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UPIPE_LIB") or os.path.join(_HERE, "libupipe.so")   # UPIPE_LIB: dev override (kernel variants)

UPIPE_UID_BYTES = 128
UPIPE_IPC_HANDLE_BYTES = 128
STATUS = {0: "UPIPE_OK", 1: "UPIPE_ERR_INVALID_ARG", 2: "UPIPE_ERR_UNSUPPORTED", 3: "UPIPE_ERR_CUDA",
          4: "UPIPE_ERR_COMM", 5: "UPIPE_ERR_WORKSPACE", 6: "UPIPE_ERR_STATE"}


class UpipeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class upipe_shape_t(ctypes.Structure):
    _fields_ = [("seq_local", c_int64), ("hidden", c_int32), ("n_q_heads", c_int32), ("n_kv_heads", c_int32),
                ("head_dim", c_int32), ("chunk_heads", c_int32), ("causal", c_int32), ("rope_base", ctypes.c_float),
                ("ring_degree", c_int32), ("qk_norm_eps", ctypes.c_float)]


class upipe_qk_norm_t(ctypes.Structure):
    _fields_ = [("q_norm_w", c_void_p), ("k_norm_w", c_void_p), ("dq_norm_w", c_void_p), ("dk_norm_w", c_void_p)]


class upipe_stage_info_t(ctypes.Structure):
    _fields_ = [("n_stages", c_int32), ("qpd", c_int32), ("kv_res", c_int32), ("sigma", c_int32),
                ("q0", c_int32), ("kv0", c_int32), ("kv_sent", c_int32)]


class upipe_comm_info_t(ctypes.Structure):
    _fields_ = [("nranks", c_int32), ("rank", c_int32), ("cuda_device", c_int32), ("transport", c_int32),
                ("max_ctas", c_int32)]


class upipe_probe_t(ctypes.Structure):
    """Test-only layout probe (include/upipe.h upipe_test_set_probe)."""
    _fields_ = [("stage", c_int32), ("q_recv", c_void_p), ("k_recv", c_void_p), ("v_recv", c_void_p),
                ("o_head", c_void_p), ("do_recv", c_void_p), ("delta_recv", c_void_p), ("dq_head", c_void_p),
                ("dk_head", c_void_p), ("dv_head", c_void_p), ("dq_recv", c_void_p), ("dk_recv", c_void_p),
                ("dv_recv", c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libupipe.so (built in-tree by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libupipe.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        st = c_int
        P = c_void_p
        sig = {
            "upipe_get_unique_id": (st, [POINTER(c_uint8)]),
            "upipe_init": (st, [POINTER(c_void_p), POINTER(c_uint8), c_int, c_int, c_int, c_uint32]),
            "upipe_fabric_create": (st, [POINTER(c_void_p), c_int]),
            "upipe_fabric_destroy": (st, [P]),
            "upipe_init_local": (st, [POINTER(c_void_p), P, c_int, c_int, c_uint32]),
            "upipe_finalize": (st, [P]),
            "upipe_status_string": (c_char_p, [c_int]),
            "upipe_last_error": (c_char_p, [P]),
            "upipe_workspace_size": (st, [c_int, POINTER(upipe_shape_t), c_int, POINTER(c_size_t)]),
            "upipe_plan_stage": (st, [c_int, POINTER(upipe_shape_t), c_int, c_int, POINTER(upipe_stage_info_t)]),
            "upipe_validate": (st, [c_int, POINTER(upipe_shape_t), c_char_p, c_size_t]),
            "upipe_attn_fwd": (st, [P, POINTER(upipe_shape_t)] + [P] * 8 + [P, c_size_t, P]),
            "upipe_attn_bwd": (st, [P, POINTER(upipe_shape_t)] + [P] * 13 + [c_int, P, c_size_t, P]),
            "upipe_attn_fwd_ex": (st, [P, POINTER(upipe_shape_t)] + [P] * 5 + [POINTER(upipe_qk_norm_t)] + [P] * 3 +
                                  [P, c_size_t, P]),
            "upipe_attn_bwd_ex": (st, [P, POINTER(upipe_shape_t)] + [P] * 5 + [POINTER(upipe_qk_norm_t)] + [P] * 8 +
                                  [c_int, P, c_size_t, P]),
            "upipe_attn_core_fwd": (st, [P] * 5 + [c_int64, c_int, c_int, c_int, c_int] + [c_int64] * 4 + [P]),
            "upipe_attn_core_bwd": (st, [P] * 9 + [c_int64, c_int, c_int, c_int, c_int] + [c_int64] * 5 + [c_int, P, P]),
            "upipe_core_bwd_sem_count": (c_int64, [c_int64, c_int]),
            "upipe_rowdot": (st, [P, c_int64, P, c_int64, P, c_int64, c_int64, c_int, c_int, P]),
            "upipe_gemm_xwT": (st, [P, P, P, c_int64, c_int64, c_int64, c_int, P]),
            "upipe_synth_fill_bf16": (st, [P, c_int64, c_uint64, c_int, c_int, c_int64, P]),
            "upipe_kernel_launches": (st, [POINTER(c_uint64)]),
            "upipe_set_trace": (st, [P, c_int]),
            "upipe_trace_read": (st, [P, POINTER(ctypes.c_double), POINTER(c_int64)]),
            "upipe_test_set_probe": (st, [P, POINTER(upipe_probe_t)]),
            "upipe_wait": (st, [P, P, c_int64]),
            "upipe_ipc_region_size": (st, [c_int, POINTER(upipe_shape_t), c_uint32, POINTER(c_size_t)]),
            "upipe_ipc_create": (st, [POINTER(c_void_p), c_int, c_int, c_int, c_uint32, POINTER(upipe_shape_t),
                                      POINTER(c_uint8)]),
            "upipe_ipc_connect": (st, [P, POINTER(c_uint8)]),
            "upipe_comm_info": (st, [P, POINTER(upipe_comm_info_t)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


EXPORTED = ("upipe_get_unique_id", "upipe_init", "upipe_fabric_create", "upipe_fabric_destroy", "upipe_init_local",
            "upipe_finalize", "upipe_status_string", "upipe_last_error", "upipe_workspace_size", "upipe_plan_stage",
            "upipe_validate", "upipe_attn_fwd", "upipe_attn_bwd", "upipe_attn_core_fwd", "upipe_attn_core_bwd", "upipe_core_bwd_sem_count",
            "upipe_rowdot", "upipe_gemm_xwT", "upipe_synth_fill_bf16", "upipe_kernel_launches", "upipe_set_trace",
            "upipe_trace_read", "upipe_test_set_probe", "upipe_wait", "upipe_comm_info",
            "upipe_ipc_region_size", "upipe_ipc_create", "upipe_ipc_connect", "upipe_attn_fwd_ex", "upipe_attn_bwd_ex")

TRACE_CATS = ("gemm", "attn_fwd", "attn_bwd", "comm", "aux")


def _check(st: int, ctx=None):
    if st != 0:
        msg = lib().upipe_last_error(ctx)
        raise UpipeError(st, msg.decode() if msg else "")


def _ptr(t):
    """Device pointer of a torch tensor (or an int / None)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def make_shape(seq_local, hidden, n_q_heads, n_kv_heads, head_dim, chunk_heads, causal=1,
               rope_base=0.0, ring_degree=0, qk_norm_eps=0.0) -> upipe_shape_t:
    return upipe_shape_t(seq_local, hidden, n_q_heads, n_kv_heads, head_dim, chunk_heads, int(causal),
                         float(rope_base), int(ring_degree), float(qk_norm_eps))


# ------------------------------------------------------------------ lifecycle

def upipe_get_unique_id() -> bytes:
    buf = (c_uint8 * UPIPE_UID_BYTES)()
    _check(lib().upipe_get_unique_id(buf))
    return bytes(buf)


def upipe_init(uid: bytes | None, cp_size: int, cp_rank: int, cuda_device: int, flags: int = 0) -> c_void_p:
    ctx = c_void_p()
    ubuf = (c_uint8 * UPIPE_UID_BYTES).from_buffer_copy(uid) if uid is not None else None
    _check(lib().upipe_init(ctypes.byref(ctx), ubuf, cp_size, cp_rank, cuda_device, flags))
    return ctx


def upipe_fabric_create(cp_size: int) -> c_void_p:
    f = c_void_p()
    _check(lib().upipe_fabric_create(ctypes.byref(f), cp_size))
    return f


def upipe_fabric_destroy(fabric) -> None:
    _check(lib().upipe_fabric_destroy(fabric))


def upipe_init_local(fabric, cp_rank: int, cuda_device: int, flags: int = 0) -> c_void_p:
    ctx = c_void_p()
    _check(lib().upipe_init_local(ctypes.byref(ctx), fabric, cp_rank, cuda_device, flags))
    return ctx


def upipe_ipc_region_size(cp_size: int, max_shape: upipe_shape_t, flags: int = 0) -> int:
    n = c_size_t()
    _check(lib().upipe_ipc_region_size(cp_size, ctypes.byref(max_shape), flags, ctypes.byref(n)))
    return n.value


def upipe_ipc_create(cp_size: int, cp_rank: int, cuda_device: int, flags: int, max_shape: upipe_shape_t):
    """Phase 1 of the direct-to-peer ctx: returns (ctx, this rank's IPC handle bytes)."""
    ctx = c_void_p()
    h = (c_uint8 * UPIPE_IPC_HANDLE_BYTES)()
    _check(lib().upipe_ipc_create(ctypes.byref(ctx), cp_size, cp_rank, cuda_device, flags, ctypes.byref(max_shape), h))
    return ctx, bytes(h)


def upipe_ipc_connect(ctx, handles: list) -> None:
    """Phase 2: handles of every rank, in rank order."""
    buf = (c_uint8 * (UPIPE_IPC_HANDLE_BYTES * len(handles))).from_buffer_copy(b"".join(handles))
    _check(lib().upipe_ipc_connect(ctx, buf), ctx)


def upipe_finalize(ctx) -> None:
    _check(lib().upipe_finalize(ctx))


def upipe_status_string(st: int) -> str:
    return lib().upipe_status_string(st).decode()


def upipe_last_error(ctx=None) -> str:
    m = lib().upipe_last_error(ctx)
    return m.decode() if m else ""


def upipe_wait(ctx, stream=None, timeout_ms: int = 0) -> None:
    """Wait for `stream` with communicator error polling; raises UpipeError (UPIPE_ERR_COMM) on a
    communicator error or timeout (the communicator is then aborted)."""
    _check(lib().upipe_wait(ctx, _stream(stream), int(timeout_ms)), ctx)


def upipe_comm_info(ctx) -> dict:
    i = upipe_comm_info_t()
    _check(lib().upipe_comm_info(ctx, ctypes.byref(i)), ctx)
    return {"nranks": i.nranks, "rank": i.rank, "cuda_device": i.cuda_device,
            "transport": {0: "none", 1: "nccl", 2: "fabric", 3: "ipc"}.get(i.transport, i.transport),
            "max_ctas": i.max_ctas}


# ------------------------------------------------------------------ planning

def upipe_workspace_size(cp_size: int, shape: upipe_shape_t, pass_: int) -> int:
    n = c_size_t()
    _check(lib().upipe_workspace_size(cp_size, ctypes.byref(shape), pass_, ctypes.byref(n)))
    return n.value


def upipe_plan_stage(cp_size: int, shape: upipe_shape_t, stage: int, device: int) -> upipe_stage_info_t:
    info = upipe_stage_info_t()
    _check(lib().upipe_plan_stage(cp_size, ctypes.byref(shape), stage, device, ctypes.byref(info)))
    return info


def upipe_validate(cp_size: int, shape: upipe_shape_t) -> tuple[int, str]:
    buf = ctypes.create_string_buffer(512)
    st = lib().upipe_validate(cp_size, ctypes.byref(shape), buf, 512)
    return st, buf.value.decode()


# ------------------------------------------------------------------ layer

def _ws_bytes(workspace, ws_bytes):
    if ws_bytes is not None:
        return ws_bytes
    return 0 if workspace is None else workspace.numel() * workspace.element_size()


def _qkn(qk_norm):
    """(q_norm_w, k_norm_w[, dq_norm_w, dk_norm_w]) -> upipe_qk_norm_t, or None."""
    if qk_norm is None:
        return None
    t = list(qk_norm) + [None] * (4 - len(qk_norm))
    return upipe_qk_norm_t(*[_ptr(a) for a in t])


def upipe_attn_fwd(ctx, shape, x, wq, wk, wv, wo, y, o_saved, lse_saved, workspace, ws_bytes=None, stream=None,
                   qk_norm=None):
    """qk_norm: (q_norm_w, k_norm_w) bf16 [d] when shape.qk_norm_eps > 0 (upipe_attn_fwd_ex)."""
    wsb = _ws_bytes(workspace, ws_bytes)
    q = _qkn(qk_norm)
    _check(lib().upipe_attn_fwd_ex(ctx, ctypes.byref(shape), _ptr(x), _ptr(wq), _ptr(wk), _ptr(wv), _ptr(wo),
                                   ctypes.byref(q) if q is not None else None, _ptr(y), _ptr(o_saved),
                                   _ptr(lse_saved), _ptr(workspace), wsb, _stream(stream)), ctx)


def upipe_attn_bwd(ctx, shape, x, wq, wk, wv, wo, dy, o_saved, lse_saved, dx, dwq, dwk, dwv, dwo, reduce_dw,
                   workspace, ws_bytes=None, stream=None, qk_norm=None):
    """qk_norm: (q_norm_w, k_norm_w, dq_norm_w, dk_norm_w) (fp32 gradients out) when shape.qk_norm_eps > 0."""
    wsb = _ws_bytes(workspace, ws_bytes)
    q = _qkn(qk_norm)
    _check(lib().upipe_attn_bwd_ex(ctx, ctypes.byref(shape), _ptr(x), _ptr(wq), _ptr(wk), _ptr(wv), _ptr(wo),
                                   ctypes.byref(q) if q is not None else None, _ptr(dy), _ptr(o_saved),
                                   _ptr(lse_saved), _ptr(dx), _ptr(dwq), _ptr(dwk), _ptr(dwv), _ptr(dwo),
                                   int(reduce_dw), _ptr(workspace), wsb, _stream(stream)), ctx)


# ------------------------------------------------------------------ kernel-level

def upipe_attn_core_fwd(q, k, v, o, lse, S, nq, nkv, d, causal, ldq, ldkv, ldo, ld_lse, stream=None):
    _check(lib().upipe_attn_core_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), S, nq, nkv, d, int(causal),
                                     ldq, ldkv, ldo, ld_lse, _stream(stream)))


CORE_ACCUMULATE, CORE_DQ_DIM_MAJOR, CORE_DETERMINISTIC = 1, 2, 4     # upipe_attn_core_bwd flags


def upipe_attn_core_bwd(q, k, v, dout, lse, delta, dq_acc, dk_acc, dv_acc, S, nq, nkv, d, causal, ldq, ldkv,
                        ldo_grad, ld_lse, ld_delta, accumulate=0, stream=None, dq_dim_major=False, dq_sem=None):
    """dq_dim_major: dq_acc is [nq*d][S]; dq_sem (zeroed int32 tensor of upipe_core_bwd_sem_count ints):
    deterministic dQ order."""
    flags = (CORE_ACCUMULATE if accumulate else 0) | (CORE_DQ_DIM_MAJOR if dq_dim_major else 0) | \
        (CORE_DETERMINISTIC if dq_sem is not None else 0)
    _check(lib().upipe_attn_core_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(dout), _ptr(lse), _ptr(delta), _ptr(dq_acc),
                                     _ptr(dk_acc), _ptr(dv_acc), S, nq, nkv, d, int(causal), ldq, ldkv, ldo_grad,
                                     ld_lse, ld_delta, flags, _ptr(dq_sem), _stream(stream)))


def upipe_core_bwd_sem_count(S: int, nq: int) -> int:
    return int(lib().upipe_core_bwd_sem_count(S, nq))


def upipe_rowdot(dO, ld_do, O, ld_o, delta, ld_delta, rows, nheads, d, stream=None):
    _check(lib().upipe_rowdot(_ptr(dO), ld_do, _ptr(O), ld_o, _ptr(delta), ld_delta, rows, nheads, d,
                              _stream(stream)))


def upipe_gemm_xwT(x, w, y, M, N, K, mode=0, stream=None):
    _check(lib().upipe_gemm_xwT(_ptr(x), _ptr(w), _ptr(y), M, N, K, mode, _stream(stream)))


def upipe_synth_fill_bf16(dst, n, seed, tensor_id, exponent, start=0, stream=None):
    _check(lib().upipe_synth_fill_bf16(_ptr(dst), n, seed, tensor_id, exponent, start, _stream(stream)))


# ------------------------------------------------------------------ instrumentation

def upipe_kernel_launches() -> int:
    n = c_uint64()
    _check(lib().upipe_kernel_launches(ctypes.byref(n)))
    return n.value


def upipe_set_trace(ctx, on: bool) -> None:
    _check(lib().upipe_set_trace(ctx, int(on)), ctx)


def upipe_trace_read(ctx) -> dict:
    """{category: (ms, count)} accumulated since the last read (waits for the events)."""
    ms = (ctypes.c_double * len(TRACE_CATS))()
    cnt = (c_int64 * len(TRACE_CATS))()
    _check(lib().upipe_trace_read(ctx, ms, cnt), ctx)
    return {k: (ms[i], cnt[i]) for i, k in enumerate(TRACE_CATS)}


# ------------------------------------------------------------------ test-only

def upipe_test_set_probe(ctx, stage: int = -1, **bufs) -> None:
    """Set (stage >= 0) or clear (stage = -1) the ctx's layout probe; bufs: torch tensors or None for the
    fields of upipe_probe_t (q_recv, k_recv, v_recv, o_head, do_recv, delta_recv, dq_head, dk_head,
    dv_head, dq_recv, dk_recv, dv_recv)."""
    names = [f for f, _ in upipe_probe_t._fields_][1:]
    unknown = set(bufs) - set(names)
    if unknown:
        raise TypeError(f"unknown probe fields {sorted(unknown)}")
    p = upipe_probe_t(stage, *[_ptr(bufs.get(n)) for n in names])
    _check(lib().upipe_test_set_probe(ctx, ctypes.byref(p)), ctx)
