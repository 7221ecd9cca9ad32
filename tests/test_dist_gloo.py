"""Multi-process host logic of the N > 1 path on CPU (gloo, world size 2).

Each rank asks the library's planner (the same code the CUDA stage loop uses) for
its stage plan, lays out integer payloads exactly as the projection epilogue
writes the all-to-all send buffer ([C][S_l][qpd*d], block p = the heads device p
owns in this stage), exchanges them with a real collective (gloo all_to_all), and
checks the received head-layout buffer bit-exactly against the oracle's
seq->head map. Also exercises the NCCL unique-id broadcast used by
UPipeAttention(process_group=...)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _payload(t_global, h, e, d):
    # 16-bit pattern = hash of the global index (token, head, element): bit-exact permutation check
    return ((t_global * 1000003 + h * 131 + e) * 2654435761) & 0xFFFF


def _worker(rank, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle
        from paper_2602_21196_b200 import upipe
        C = WORLD
        S_l, D, Hq, Hkv, d = 24, 64, 8, 2, 64
        for U in (2, 4, 8):
            sh = upipe.make_shape(S_l, D, Hq, Hkv, d, U)
            info0 = upipe.upipe_plan_stage(C, sh, 0, 0)
            stages = oracle.gqa_schedule(Hq, Hkv, C, U)
            assert info0.n_stages == len(stages)
            for s in range(info0.n_stages):
                plans = [upipe.upipe_plan_stage(C, sh, s, p) for p in range(C)]
                qpd = plans[0].qpd
                # send layout of this rank: block p = [S_l][qpd*d] for device p's heads
                send = np.zeros((C, S_l, qpd * d), dtype=np.int64)
                for p in range(C):
                    for j in range(qpd):
                        h = plans[p].q0 + j
                        for t in range(S_l):
                            send[p, t, j * d:(j + 1) * d] = _payload(rank * S_l + t, h, np.arange(d), d)
                recv = torch.empty(C * S_l * qpd * d, dtype=torch.int64)
                dist.all_to_all_single(recv, torch.from_numpy(send.reshape(-1)))
                got = recv.numpy().reshape(C * S_l, qpd, d)     # [S][qpd][d] head layout
                # oracle map: device `rank` gets the full sequence of its stage heads
                heads = stages[s].q_heads
                shards = [{h: np.stack([_payload(r * S_l + t, h, np.arange(d), d) for t in range(S_l)])
                           for p in range(C) for h in heads[p]} for r in range(C)]
                want = oracle.a2a_seq_to_head(shards, heads)[rank]
                assert np.array_equal(got, want), (U, s)
        # the uid broadcast of UPipeAttention(process_group=...)
        obj = [upipe.upipe_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert isinstance(obj[0], bytes) and len(obj[0]) == upipe.UPIPE_UID_BYTES
        # max-over-ranks timing reduction used by bench.py
        t = torch.tensor([10.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == 11.0
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_gloo_world2_a2a_layout_and_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for r, msg in res:
        assert msg == "ok", f"rank {r}: {msg}"
