"""Direct-to-peer transport run as C separate PROCESSES, all on cuda:0: every rank
maps the others' symmetric regions with CUDA IPC and pushes its blocks straight into their receive
buffers (ready / done flags written and waited on by the GPU front end). The gloo process group only
exchanges the IPC handles; no NCCL is involved. This is the library's stage loop running across
processes, checked against the un-sharded fp64 oracle at the north_star bar, and bitwise against the
single-process fabric (forward; the backward in deterministic mode)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth
from test_gpu_layer import ABS, _boundary_abs, _check, _run_group

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, C, port, cfg, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), UPIPE_QUIET="1")
    dist.init_process_group("gloo", rank=rank, world_size=C)
    torch.cuda.set_device(0)
    from paper_2602_21196_b200 import UPipeAttention
    S, D, Hq, Hkv, d, U = cfg["S"], cfg["D"], cfg["Hq"], cfg["Hkv"], cfg["d"], cfg["U"]
    inp = synth.layer_inputs(0, S, D, Hq, Hkv, d)
    S_l = S // C
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).to(dev)  # noqa: E731
    W = [t(inp[k]) for k in ("wq", "wk", "wv", "wo")]
    x, dy = t(inp["x"][rank * S_l:(rank + 1) * S_l]), t(inp["dy"][rank * S_l:(rank + 1) * S_l])
    attn = UPipeAttention(Hq, Hkv, d, D, U, True, process_group=dist.group.WORLD, transport="ipc",
                          max_seq_local=S_l, sync_comm=cfg.get("sync", False), ring_degree=cfg.get("ring", 1),
                          deterministic=cfg.get("det", False), direct=cfg.get("direct", False),
                          rope_base=cfg.get("rope", 0.0), qk_norm_eps=cfg.get("qkn", 0.0))
    NW = {}
    if cfg.get("qkn"):
        NW = dict(q_norm_w=t(synth.norm_weight(0, "q_norm_w", d)), k_norm_w=t(synth.norm_weight(0, "k_norm_w", d)))
    info = attn.comm_info()
    assert info["transport"] == "ipc" and info["nranks"] == C and info["rank"] == rank, info
    y, saved = attn.forward(x, *W, **NW)
    g = attn.backward(x, *W, dy, saved, **NW)
    attn.wait(timeout_s=300)
    out = {"y": y, "o": saved[0], "lse": saved[1], "dx": g[0], "dwq": g[1], "dwk": g[2], "dwv": g[3], "dwo": g[4]}
    if NW:
        out.update(dgq=g[5], dgk=g[6])
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **{k: v.float().cpu().numpy() for k, v in out.items()},
             region=np.array([attn.region_bytes]))
    attn.close()
    dist.barrier()
    dist.destroy_process_group()


def _run_ipc(C, cfg):
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_rank, args=(C, _free_port(), cfg, td), nprocs=C, join=True, start_method="spawn")
        res = [dict(np.load(os.path.join(td, f"r{r}.npz"))) for r in range(C)]
    return [{k: torch.from_numpy(v) for k, v in r.items()} for r in res]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("C,S,D,Hq,Hkv,d,U,sync,ring", [
    (2, 512, 512, 8, 2, 64, 2, False, 1),       # BASELINE configs[0] schedule, overlapped
    (2, 512, 512, 8, 2, 64, 2, True, 1),        # sequential (one buffer set)
    (4, 1024, 1024, 32, 8, 128, 8, False, 1),   # Llama3-8B heads at CP 4, U 8 (qpd 2, sigma 2)
    (4, 1024, 512, 16, 4, 64, 16, False, 1),    # Ulysses (U = Hq)
    (4, 1024, 512, 8, 2, 64, 2, True, 2),       # ring hybrid (2 x 2): ring steps as IPC send/recv
])
def test_ipc_multiprocess_layer_matches_oracle(C, S, D, Hq, Hkv, d, U, sync, ring):
    cfg = dict(S=S, D=D, Hq=Hq, Hkv=Hkv, d=d, U=U, sync=sync, ring=ring)
    res = _run_ipc(C, cfg)
    inp = synth.layer_inputs(0, S, D, Hq, Hkv, d)
    _check(res, inp, C, Hq, Hkv, d, U, ring=ring)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("C,S,D,Hq,Hkv,d,U,rope,ring", [
    (2, 512, 512, 8, 2, 64, 2, 0.0, 1),         # BASELINE configs[0] schedule
    (4, 1024, 1024, 32, 8, 128, 8, 0.0, 1),     # Llama3-8B heads at CP 4, U 8 (qpd 2, sigma 2)
    (8, 1024, 1024, 32, 8, 128, 8, 5e5, 1),     # Llama3-8B heads at CP 8, U 8 (qpd 1, sigma 4), RoPE
    (4, 1024, 512, 16, 4, 64, 16, 0.0, 1),      # Ulysses (U = Hq)
    (4, 1000, 512, 16, 16, 64, 8, 0.0, 1),      # MHA, ragged S_l = 250 (tiles straddle the rank blocks)
    (4, 1024, 512, 8, 2, 64, 2, 1e4, 2),        # UPipe x Ring (2 x 2): direct Ulysses all-to-alls, IPC ring steps
])
def test_ipc_direct_layer_matches_oracle(C, S, D, Hq, Hkv, d, U, rope, ring):
    # UPIPE_FLAG_DIRECT: the projection / dO epilogues, the attention epilogues (O, dK, dV) and the
    # dQ conversion store straight into the owners' receive buffers in the other processes
    res = _run_ipc(C, dict(S=S, D=D, Hq=Hq, Hkv=Hkv, d=d, U=U, direct=True, rope=rope, ring=ring))
    inp = synth.layer_inputs(0, S, D, Hq, Hkv, d)
    _check(res, inp, C, Hq, Hkv, d, U, rope_base=rope or None, ring=ring)


@pytest.mark.timeout(900)
def test_ipc_direct_qk_norm_matches_oracle():
    # N2 direct stores with the Qwen3 q/k norm (N3): the fused norm backward writes dQ / dK into the peers
    C, S, D, Hq, Hkv, d, U = 4, 1024, 1024, 64, 8, 128, 8
    res = _run_ipc(C, dict(S=S, D=D, Hq=Hq, Hkv=Hkv, d=d, U=U, direct=True, rope=1e6, qkn=1e-6))
    inp = synth.layer_inputs(0, S, D, Hq, Hkv, d)
    inp.update(q_norm_w=synth.norm_weight(0, "q_norm_w", d), k_norm_w=synth.norm_weight(0, "k_norm_w", d),
               qk_norm_eps=1e-6)
    eo, ey = _boundary_abs(inp, Hq, Hkv, d, 1e6)
    _check(res, inp, C, Hq, Hkv, d, U, rope_base=1e6, abs_y=max(ABS, ey), abs_o=max(ABS, eo))


@pytest.mark.timeout(900)
def test_ipc_direct_equals_fabric_bitwise_deterministic():
    # the direct-to-peer stores move exactly the bytes the fabric's all-to-alls move: bitwise equal outputs
    # (deterministic backward), and the symmetric region holds no send buffers
    C, S, D, Hq, Hkv, d, U = 4, 1024, 512, 16, 4, 64, 4
    res = _run_ipc(C, dict(S=S, D=D, Hq=Hq, Hkv=Hkv, d=d, U=U, det=True, direct=True))
    fab, _ = _run_group(C, S, D, Hq, Hkv, d, U, det=True)
    for p in range(C):
        for k in ("y", "o", "lse", "dx", "dwq", "dwk", "dwv", "dwo"):
            a = res[p][k].float()
            b = fab[p][k].float().cpu()
            assert torch.equal(a, b), (p, k, (a - b).abs().max().item())
    plain = _run_ipc(C, dict(S=S, D=D, Hq=Hq, Hkv=Hkv, d=d, U=U, det=True, sync=True))
    assert int(res[0]["region"][0]) < int(plain[0]["region"][0])


@pytest.mark.timeout(900)
def test_ipc_equals_fabric_bitwise_deterministic():
    # same kernels, same per-rank inputs: the IPC processes and the single-process fabric threads give
    # bitwise identical outputs in deterministic mode (the transport only moves bytes)
    C, S, D, Hq, Hkv, d, U = 4, 1024, 512, 16, 4, 64, 4
    res = _run_ipc(C, dict(S=S, D=D, Hq=Hq, Hkv=Hkv, d=d, U=U, det=True))
    fab, _ = _run_group(C, S, D, Hq, Hkv, d, U, det=True)
    for p in range(C):
        for k in ("y", "o", "lse", "dx", "dwq", "dwk", "dwv", "dwo"):
            a = res[p][k].float()
            b = fab[p][k].float().cpu()
            assert torch.equal(a, b), (p, k, (a - b).abs().max().item())
