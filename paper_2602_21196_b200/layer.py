"""User-facing wrapper of the UPipe layer: owns a libupipe context and the
workspace (allocated from the PyTorch caching allocator so it shows up in
``torch.cuda.max_memory_allocated``). Marshalling only; the math runs in libupipe.

    attn = UPipeAttention(n_q_heads=32, n_kv_heads=8, head_dim=128, hidden=4096,
                          chunk_heads=8, process_group=pg)      # CP group = pg
    y, saved = attn.forward(x_shard, wq, wk, wv, wo)
    dx, dwq, dwk, dwv, dwo = attn.backward(x_shard, wq, wk, wv, wo, dy, saved)
"""
from __future__ import annotations

import torch

from . import upipe as U


class UPipeAttention:
    def __init__(self, n_q_heads: int, n_kv_heads: int, head_dim: int, hidden: int, chunk_heads: int,
                 causal: bool = True, process_group=None, device=None, fabric=None, cp_rank: int | None = None,
                 cp_size: int | None = None, sync_comm: bool = False, naive_kv: bool = False,
                 rope_base: float = 0.0, ring_degree: int = 1, deterministic: bool = False,
                 transport: str = "nccl", max_seq_local: int | None = None, direct: bool = False,
                 qk_norm_eps: float = 0.0):
        """CP group: ``process_group`` (torch.distributed, one process per GPU, NCCL transport),
        or ``fabric`` + ``cp_rank`` + ``cp_size`` (single-process group driven by one host thread per rank),
        or neither (C = 1). ``sync_comm``: sequential schedule with one chunk buffer set (the
        paper's memory-minimal form); default overlaps the next chunk's all-to-all with the current
        chunk's attention on a side stream (two buffer sets). ``ring_degree`` r > 1: UPipe x Ring hybrid
        (DESIGN A27): Ulysses groups of C/r consecutive ranks, Ring Attention across the r groups.
        ``deterministic``: bitwise-reproducible backward (dQ partials added in key-tile order; slower).
        ``transport="ipc"`` (with ``process_group`` and ``max_seq_local``): direct-to-peer all-to-alls over
        CUDA IPC peer memory instead of NCCL; the handles are exchanged over the group (any
        backend, gloo included), the library owns the symmetric workspace (sized for ``max_seq_local``).
        ``direct`` (with ``transport="ipc"``, UPIPE_FLAG_DIRECT): the all-to-alls are fused into their
        producers -- projection / attention / dQ-conversion epilogues store straight into the owners'
        receive buffers, no send buffers.
        ``qk_norm_eps`` > 0: Qwen3 per-head RMSNorm of Q and K (DESIGN A29); ``forward`` then takes
        ``q_norm_w``, ``k_norm_w`` (bf16 [head_dim]) and ``backward`` returns their fp32 gradients too."""
        self.Hq, self.Hkv, self.d, self.D, self.U = n_q_heads, n_kv_heads, head_dim, hidden, chunk_heads
        self.ipc = False
        self.region_bytes = 0
        self.causal = int(causal)
        self.rope_base = float(rope_base)    # 0: no RoPE; else rotary base (Llama3: 500000), DESIGN A26
        self.ring = max(1, int(ring_degree))
        self.qk_norm_eps = float(qk_norm_eps)
        # UPIPE_FLAG_SYNC_COMM, UPIPE_FLAG_NAIVE_KV, UPIPE_FLAG_DETERMINISTIC
        # UPIPE_FLAG_DIRECT (8): direct-to-peer all-to-alls fused into the producing kernels (IPC only)
        if direct and transport != "ipc":
            raise ValueError("direct=True needs transport='ipc' (peer memory)")
        self.flags = (1 if sync_comm else 0) | (2 if naive_kv else 0) | (4 if deterministic else 0) | \
            (8 if direct else 0)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        if fabric is not None:
            self.C = cp_size
            self.ctx = U.upipe_init_local(fabric, cp_rank, dev_index, self.flags)
            self.rank = cp_rank
        elif process_group is not None and transport == "ipc":
            import torch.distributed as dist
            if max_seq_local is None:
                raise ValueError("transport='ipc' needs max_seq_local (the symmetric region is sized once)")
            self.C = dist.get_world_size(process_group)
            self.rank = dist.get_rank(process_group)
            self.ctx, h = U.upipe_ipc_create(self.C, self.rank, dev_index, self.flags, self.shape(max_seq_local))
            handles = [None] * self.C
            dist.all_gather_object(handles, h, group=process_group)
            U.upipe_ipc_connect(self.ctx, handles)
            self.ipc = True
            self.region_bytes = U.upipe_ipc_region_size(self.C, self.shape(max_seq_local), self.flags)
        elif process_group is not None:
            import torch.distributed as dist
            self.C = dist.get_world_size(process_group)
            self.rank = dist.get_rank(process_group)
            obj = [U.upipe_get_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(process_group, 0), group=process_group)
            self.ctx = U.upipe_init(obj[0], self.C, self.rank, dev_index, self.flags)
        else:
            self.C, self.rank = 1, 0
            self.ctx = U.upipe_init(None, 1, 0, dev_index, self.flags)
        self._ws = {}

    def shape(self, seq_local: int) -> U.upipe_shape_t:
        return U.make_shape(seq_local, self.D, self.Hq, self.Hkv, self.d, self.U, self.causal, self.rope_base,
                            self.ring, self.qk_norm_eps)

    def workspace(self, seq_local: int, pass_: int) -> torch.Tensor:
        # One chunk-buffer workspace per sequence length, shared by the forward and the backward pass
        # (they never run at the same time and nothing in it outlives a call): sized for the larger.
        key = seq_local
        if key not in self._ws:
            sync = 2 if self.flags & 1 else 0
            naive = 8 if self.flags & 2 else 0
            n = max(U.upipe_workspace_size(self.C, self.shape(seq_local), p + sync + naive) for p in (0, 1))
            self._ws[key] = torch.empty(max(n, 256), dtype=torch.uint8, device=self.device)
        return self._ws[key]

    def release_workspace(self):
        self._ws.clear()

    def _norm_w(self, q_norm_w, k_norm_w):
        if self.qk_norm_eps > 0 and (q_norm_w is None or k_norm_w is None):
            raise ValueError("qk_norm_eps > 0: pass q_norm_w and k_norm_w")
        return (q_norm_w, k_norm_w) if self.qk_norm_eps > 0 else None

    def forward(self, x, wq, wk, wv, wo, stream=None, q_norm_w=None, k_norm_w=None):
        S_l = x.shape[0]
        sh = self.shape(S_l)
        y = torch.empty((S_l, self.D), dtype=torch.bfloat16, device=x.device)
        o_saved = torch.empty((S_l, self.Hq * self.d), dtype=torch.bfloat16, device=x.device)
        a = self.C // self.ring                  # Ulysses degree; lse covers the rank's heads over its group's tokens
        lse = torch.empty((self.Hq // a, S_l * a), dtype=torch.float32, device=x.device)
        ws = None if self.ipc else self.workspace(S_l, 0)     # IPC: the library's symmetric region
        U.upipe_attn_fwd(self.ctx, sh, x, wq, wk, wv, wo, y, o_saved, lse, ws, stream=stream,
                         qk_norm=self._norm_w(q_norm_w, k_norm_w))
        return y, (o_saved, lse)

    def backward(self, x, wq, wk, wv, wo, dy, saved, reduce_dw: bool = True, stream=None, q_norm_w=None,
                 k_norm_w=None):
        o_saved, lse = saved
        S_l = x.shape[0]
        sh = self.shape(S_l)
        dx = torch.empty_like(x)
        dwq = torch.empty(wq.shape, dtype=torch.float32, device=x.device)
        dwk = torch.empty(wk.shape, dtype=torch.float32, device=x.device)
        dwv = torch.empty(wv.shape, dtype=torch.float32, device=x.device)
        dwo = torch.empty(wo.shape, dtype=torch.float32, device=x.device)
        ws = None if self.ipc else self.workspace(S_l, 1)
        nw = self._norm_w(q_norm_w, k_norm_w)
        if nw is None:
            U.upipe_attn_bwd(self.ctx, sh, x, wq, wk, wv, wo, dy, o_saved, lse, dx, dwq, dwk, dwv, dwo, reduce_dw, ws,
                             stream=stream)
            return dx, dwq, dwk, dwv, dwo
        dgq = torch.empty(self.d, dtype=torch.float32, device=x.device)
        dgk = torch.empty(self.d, dtype=torch.float32, device=x.device)
        U.upipe_attn_bwd(self.ctx, sh, x, wq, wk, wv, wo, dy, o_saved, lse, dx, dwq, dwk, dwv, dwo, reduce_dw, ws,
                         stream=stream, qk_norm=(nw[0], nw[1], dgq, dgk))
        return dx, dwq, dwk, dwv, dwo, dgq, dgk

    def wait(self, timeout_s: float = 0.0, stream=None):
        """Block until this rank's enqueued layer work is done, failing (UpipeError, communicator aborted)
        on a communicator error or after ``timeout_s`` seconds without completion (a dead peer)."""
        U.upipe_wait(self.ctx, stream, int(timeout_s * 1000))

    def comm_info(self) -> dict:
        return U.upipe_comm_info(self.ctx)

    def close(self):
        if self.ctx is not None:
            U.upipe_finalize(self.ctx)
            self.ctx = None
        self._ws.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
