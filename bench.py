#!/usr/bin/env python
"""UPipe layer benchmark (contract: DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: one rank per GPU, NCCL)

One step = one UPipe attention layer forward + backward (all SURVEY §8a rows:
projections, seq->head all-to-all, causal GQA attention, head->seq all-to-all,
output projection, and the backward of each) over the whole sequence, on the
Llama3-8B attention shape (32 Q / 8 KV heads, d=128, hidden 4096), S = 131072
tokens (BASELINE configs[1]), context-parallel degree C = N, chunk U = 8.
Inputs are synthetic (the seeded counter-based generator, drawn on the device)
and larger than L2, so no flush is needed between steps. Rank 0 prints one JSON line.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Llama3-8B attn fwd+bwd tokens/s/GPU & peak activation GB at 1/2/4/8 B200"
LLAMA = dict(Hq=32, Hkv=8, d=128, D=4096)
MODELS = {   # BASELINE configs: Llama3-8B attention (configs 1-4) and the 32B-class GQA layer (config 5)
    "llama3-8b": dict(LLAMA, name="Llama3-8B attention layer", workload="llama3-8b-attention-layer-fwd-bwd"),
    "32b": dict(Hq=64, Hkv=8, d=128, D=5120, name="32B-class GQA attention layer (64Q/8KV, d=128, hidden 5120)",
                workload="32b-gqa-attention-layer-fwd-bwd"),
}


def a2a_bytes(S_l, C, Hq, Hkv, d, U, naive=False):
    """Bytes ONE rank sends to the other C - 1 ranks in one layer fwd+bwd, from the GQA schedule's buffer sizes
    (Table 4): forward Q and O per stage, K and V per super-stage (every stage when
    naive); backward Q, dO, dQ (bf16) and delta (fp32) per stage, K, V, dK, dV per super-stage. Each chunk
    keeps 1/C of its blocks on the rank. Returns {"fwd_inp", "fwd_out", "bwd", "total"}."""
    qpd, R = U // C, Hq // Hkv
    kv_res = max(1, qpd // R)
    sigma = 1 if naive else max(1, R // qpd)
    stages = Hq // U
    kv_events = stages // sigma
    off = (C - 1) / C
    qb = S_l * qpd * d * 2 * C                   # one Q-sized chunk (C blocks of [S_l][qpd d] bf16)
    kb = S_l * kv_res * d * 2 * C
    fwd_inp = (stages * qb + kv_events * 2 * kb) * off
    fwd_out = stages * qb * off
    bwd = (stages * (3 * qb + S_l * qpd * 4 * C) + kv_events * 4 * kb) * off
    return {"fwd_inp": fwd_inp, "fwd_out": fwd_out, "bwd": bwd, "total": fwd_inp + fwd_out + bwd}


def memory_by_cp(upipe, S, Hq, Hkv, d, D, U, naive=False):
    """Per-rank chunk buffers at the metric's CP degrees 1/2/4/8 for this S and U, from the library's workspace
    planner (exact byte counts of the buffers the library would use; host-side, so the 2/4/8-GPU points are
    PLANNED, not measured on this one-GPU run): the overlapped schedule (default for C > 1), the sequential one
    and the direct-to-peer one (N2), UPipe against chunk = all-heads Ulysses. Chunk buffers = workspace minus
    the U-independent gradient buffer (DESIGN A21, A30)."""
    out = {}
    gib = float(2 ** 30)
    for C in (1, 2, 4, 8):
        if S % C or U % C or Hkv % C:
            continue
        S_l = S // C
        g = S_l * min((Hq + 2 * Hkv) * d * 2, D * 4) if not naive else S_l * D * 4
        row = {}
        for name, (pf, pb) in (("overlap", (0, 1)), ("sequential", (2, 3)), ("direct", (4, 5))):
            if C == 1 and name != "sequential":
                continue
            nv = 8 if naive else 0
            sh_u = upipe.make_shape(S_l, D, Hq, Hkv, d, U)
            sh_h = upipe.make_shape(S_l, D, Hq, Hkv, d, Hq)
            up = [upipe.upipe_workspace_size(C, sh_u, p + nv) for p in (pf, pb)]
            ul = [upipe.upipe_workspace_size(C, sh_h, p + nv) for p in (pf, pb)]
            up_chunk = max(up[0], up[1] - (g if Hq // U > 1 else 0))
            ul_chunk = max(ul[0], ul[1])
            row[name] = {"workspace_gib": max(up) / gib, "chunk_buffers_gib": up_chunk / gib,
                         "ulysses_chunk_buffers_gib": ul_chunk / gib, "reduction": 1 - up_chunk / ul_chunk}
        out[str(C)] = row
    out["note"] = "per rank, from upipe_workspace_size (planned; only C = N is measured by this run)"
    return out


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--seq", type=int, default=131072, help="global sequence length S")
    ap.add_argument("--chunk", type=int, default=8, help="chunk_heads U (UPipe); Ulysses = 32")
    ap.add_argument("--rope-base", type=float, default=0.0,
                    help="RoPE on Q/K with this base (Llama3: 500000; SURVEY N3); 0 = off (north_star layer)")
    ap.add_argument("--naive-kv", action="store_true",
                    help="ablation (SURVEY N1): re-send K/V every stage instead of once per GQA super-stage")
    ap.add_argument("--model", choices=sorted(MODELS), default="llama3-8b",
                    help="layer shape (default: BASELINE's headline Llama3-8B layer)")
    ap.add_argument("--ring", type=int, default=1,
                    help="ring degree r of the UPipe x Ring hybrid (N > 1: Ulysses groups of N/r ranks; SURVEY N4)")
    ap.add_argument("--no-ulysses", action="store_true", help="skip the chunk=all-heads Ulysses comparison")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quick", action="store_true", help="profiling runs: timed region only")
    ap.add_argument("--qk-norm", type=float, default=0.0,
                    help="Qwen3 per-head q/k RMSNorm with this eps (1e-6; SURVEY N3, DESIGN A29); 0 = off")
    ap.add_argument("--transport", choices=["nccl", "ipc"], default="nccl",
                    help="N > 1: NCCL collectives, or CUDA-IPC peer memory (the library's symmetric region)")
    ap.add_argument("--direct", action="store_true",
                    help="with --transport ipc: all-to-alls fused into their producers (UPIPE_FLAG_DIRECT, SURVEY N2)")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------- peaks / clocks

def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"bf16_burst": j["bf16_tflops"], "bf16_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                "hbm": j["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_burst": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows)
        mx = max(float(r[2]) for r in rows)
        load = [float(r[1]) for r in rows if float(r[3]) > 200.0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        load.sort()
        return {"sm_mhz": load[len(load) // 2], "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows)}


# ----------------------------------------------------------------------------- FLOP model

def causal_pairs(S):
    return S * (S + 1) // 2


def flops_attn_bwd_per_head(S, d, causal=True):
    """5 matmuls (S^T, dP^T, dV, dK, dQ) x 2 flops x d per visible (query, key) pair."""
    pairs = causal_pairs(S) if causal else S * S
    return 10.0 * d * pairs


def flops_step_per_rank(S, C, Hq, Hkv, d, D, causal=True):
    pairs = causal_pairs(S) if causal else S * S
    attn = 14.0 * d * pairs * Hq / C                 # fwd 4 d + bwd 10 d per pair and head
    proj = 6.0 * (S / C) * D * d * (2 * Hq + 2 * Hkv)  # Q,K,V,O forward (2x) + backward (4x)
    return attn + proj


# ----------------------------------------------------------------------------- oracle (CPU) legs

def oracle_step_time(S, shape=LLAMA, seed=0):
    """One oracle fwd+bwd of the Llama-shaped layer at sequence length S on the host cores."""
    import numpy as np  # noqa: F401
    import oracle
    import synth
    inp = synth.layer_inputs(seed, S, shape["D"], shape["Hq"], shape["Hkv"], shape["d"])
    args = [inp[k] for k in ("x", "wq", "wk", "wv", "wo")]
    t0 = time.perf_counter()
    oracle.layer_fwd(*args, shape["Hq"], shape["Hkv"], shape["d"])
    oracle.layer_bwd(*args, inp["dy"], shape["Hq"], shape["Hkv"], shape["d"])
    return time.perf_counter() - t0


def cpu_cores():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        n = max((i.get("num_threads", 1) for i in info), default=os.cpu_count())
        return int(n)
    except Exception:
        return os.cpu_count()


def cpu_baseline(budget_s=20.0):
    """Oracle timed on a bounded sample of the workload (Llama3-8B layer shape, smaller S)."""
    S = 1024
    t = oracle_step_time(S)
    while t * 3.5 < budget_s / 2 and S < 8192:    # attention ~S^2, projections ~S: grow while cheap
        S *= 2
        t = oracle_step_time(S)
    return {"value": S / t, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
            "sample": f"one fp64 numpy oracle fwd+bwd of the Llama3-8B attention layer (32Q/8KV, d=128, D=4096) "
                      f"at S={S} tokens (un-sharded), {t:.2f} s; tokens/s = S / t at that S (cost grows ~S^2)",
            "seconds": t, "S": S}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    S = 1024
    oracle_step_time(256)           # import / first-touch warm-up
    for _ in range(args.warmup):
        oracle_step_time(S)
    ts = [oracle_step_time(S) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    v = S / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s/GPU", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "llama3-8b-attention-layer-fwd-bwd", "seq_len": S, "global_batch": 1,
                       "parallelism": "none (host cores)", "note": "bounded sample of the bench workload"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": f"oracle fwd+bwd, Llama3-8B layer shape at S={S} per step"},
            "e2e": {"value": v, "unit": "tokens/s/GPU", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    # UPIPE_BENCH_SAME_GPU=1 (tests only): every rank on cuda:0 with a gloo process group, so the N > 1 code
    # path (IPC transport, max-over-ranks timing, all-to-all accounting) runs on a one-GPU box; its timings
    # are of ranks sharing one GPU and mean nothing
    same_gpu = os.environ.get("UPIPE_BENCH_SAME_GPU") == "1"
    if same_gpu and world > 1 and args.transport != "ipc":
        raise SystemExit("UPIPE_BENCH_SAME_GPU=1 needs --transport ipc (NCCL cannot run two ranks on one GPU)")
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    from paper_2602_21196_b200 import UPipeAttention, upipe
    import synth

    C = world
    M = MODELS[args.model]
    Hq, Hkv, d, D = M["Hq"], M["Hkv"], M["d"], M["D"]
    S = args.seq
    assert S % C == 0
    S_l = S // C
    U = args.chunk
    e = synth.layer_exponents(D, Hq, d, S)

    def fill(shape, name, start=0):
        t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        upipe.upipe_synth_fill_bf16(t, t.numel(), 0, synth.TID[name], e[name], start)
        return t

    x = fill((S_l, D), "x", rank * S_l * D)
    dy = fill((S_l, D), "dy", rank * S_l * D)
    W = [fill((Hq * d, D), "wq"), fill((Hkv * d, D), "wk"), fill((Hkv * d, D), "wv"), fill((D, Hq * d), "wo")]
    NW = {}                                        # Qwen3 q/k norm weights (DESIGN A29)
    if args.qk_norm > 0:
        NW = {k: torch.from_numpy(synth.norm_weight(0, k, d).astype("float32")).to(torch.bfloat16).to(dev)
              for k in ("q_norm_w", "k_norm_w")}
    torch.cuda.synchronize()

    def make_attn(chunk):
        kw = {}
        if pg is not None and args.transport == "ipc":
            kw = dict(transport="ipc", max_seq_local=S_l, direct=args.direct)
        return UPipeAttention(Hq, Hkv, d, D, chunk, True, process_group=pg, naive_kv=args.naive_kv,
                              rope_base=args.rope_base, ring_degree=args.ring, qk_norm_eps=args.qk_norm, **kw)

    def barrier():
        if pg is not None:
            dist.barrier()

    def max_over_ranks(v):
        if pg is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if same_gpu else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def run(chunk, steps, warmup, trace=False):
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()       # inputs and weights only: workspace + outputs count as activation
        attn = make_attn(chunk)
        out = {}

        def step():
            y, saved = attn.forward(x, *W, **NW)
            g = attn.backward(x, *W, dy, saved, **NW)
            return y, g

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        step()
        torch.cuda.synchronize()
        out["peak_bytes"] = max_over_ranks(torch.cuda.max_memory_allocated() - base)   # max over ranks
        out["ws_bytes"] = attn.region_bytes if attn.ipc else sum(t.numel() for t in attn._ws.values())
        # chunk buffers = workspace minus the U-independent pre-allocated gradient buffer G [S_l, (Hq + 2 Hkv) d]
        # bf16 (DESIGN A30; with --naive-kv the fp32 dX accumulator [S_l, D], only with more than one stage):
        # the "intermediate tensors" of P:332-343 (DESIGN A21)
        fixed = 0
        if Hq // chunk > 1:
            gb = (Hq + 2 * Hkv) * d * 2
            fixed = S_l * (D * 4 if args.naive_kv or gb > D * 4 else gb)
        out["chunk_bytes"] = out["ws_bytes"] - fixed
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if trace:
            upipe.upipe_set_trace(attn.ctx, True)
            upipe.upipe_trace_read(attn.ctx)
        barrier()
        torch.cuda.synchronize()
        l0 = upipe.upipe_kernel_launches()
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        l1 = upipe.upipe_kernel_launches()
        barrier()
        out["ms"] = max_over_ranks(e0.elapsed_time(e1))
        out["launches"] = l1 - l0
        if trace:
            out["trace"] = upipe.upipe_trace_read(attn.ctx)
            upipe.upipe_set_trace(attn.ctx, False)
        out["attn"] = attn
        return out

    sampler = ClockSampler(local) if local == 0 and rank == 0 else None
    if sampler:
        sampler.start()
    main_run = run(U, args.steps, args.warmup, trace=True)
    clocks = sampler.stop() if sampler else None
    ms_step = main_run["ms"] / args.steps
    tok_s_total = S * args.steps / (main_run["ms"] / 1e3)    # the whole job (all C ranks share one sequence)
    tok_s = tok_s_total / world                                # the metric: tokens/s/GPU (P:388 normalisation)

    # roofline of the dominant kernel (attention backward), timed live by the in-library trace events
    peaks = measured_peaks()
    tr = main_run["trace"]
    bwd_ms, bwd_n = tr["attn_bwd"]
    a_deg = C // args.ring                          # Ulysses degree (C unless the ring hybrid is on)
    qpd = U // a_deg
    if args.ring == 1:
        flops_bwd_launch = flops_attn_bwd_per_head(S, d) * qpd
    else:
        # ring hybrid, this rank (ring block i = rank // a): per stage its own causal block plus i full
        # blocks of S_b = S / r keys; report the mean over those launches
        S_b, ring_i = S // args.ring, rank // a_deg
        flops_bwd_launch = 10.0 * d * qpd * (causal_pairs(S_b) + ring_i * S_b * S_b) / (1 + ring_i)
    achieved = flops_bwd_launch / (bwd_ms / bwd_n / 1e3) / 1e12 if bwd_n else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "attn_bwd_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            j = json.load(f)
        if j.get("seq") == S and j.get("chunk") == U and j.get("C") == C and j.get("model", "llama3-8b") == args.model:
            traffic = j.get("dram_bytes_per_launch")
    step_flops = flops_step_per_rank(S, C, Hq, Hkv, d, D)
    per_step_ms = {k: v[0] / args.steps for k, v in tr.items()}

    result = {
        "metric": METRIC, "value": tok_s, "unit": "tokens/s/GPU", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded counter-based generator, drawn on device)",
        "config": {"workload": M["workload"] + (" (BASELINE configs[1])" if args.model == "llama3-8b" and S == 131072 else ""),
                   "model": M["name"],
                   "n_q_heads": Hq, "n_kv_heads": Hkv, "head_dim": d, "hidden": D, "seq_len": S, "global_batch": 1,
                   "chunk_heads": U, "cp": C,
                   "parallelism": f"cp{C} (UPipe, U={U})" if args.ring == 1 else
                   f"cp{C} = ulysses{C // args.ring} x ring{args.ring} (UPipe x Ring, U={U})",
                   "kv_schedule": "naive (per-stage K/V resend)" if args.naive_kv else "GQA super-stage (P:362-380)",
                   "rope_base": args.rope_base, "qk_norm_eps": args.qk_norm,
                   "transport": ("ipc-direct" if args.direct else args.transport) if C > 1 else "none (C = 1)",
                   "l2": f"inputs larger than L2 (x, dy: S_l x {D} bf16 per rank); no flush needed"},
        "tokens_per_s_total": tok_s_total,
        "value_definition": "S / (C * max-over-ranks device time of one fwd+bwd step): tokens/s/GPU as BASELINE's "
                            "metric names it; tokens_per_s_total = S / time",
        "gpu_launches": main_run["launches"],
        "gpu_launches_per_step": main_run["launches"] / args.steps,
        "roofline": {"kernel": "attn_bwd (tcgen05 flash attention backward)", "bound": "tensor",
                     "achieved": achieved, "peak": peaks["bf16_sustained"], "unit": "TFLOP/s",
                     "frac": (achieved / peaks["bf16_sustained"]) if achieved else None, "traffic": traffic,
                     "peak_source": peaks["source"] + ", bf16 sustained (kernel timed inside a long step)",
                     "flops_per_launch": flops_bwd_launch, "launches": bwd_n,
                     "avg_launch_ms": bwd_ms / bwd_n if bwd_n else None,
                     "per_unit": "10*d flops per causal (query,key) pair per head; launch = qpd heads x S(S+1)/2 pairs"},
        "step_roofline": {"flops_per_step_per_rank": step_flops,
                          "achieved_tflops": step_flops / (ms_step / 1e3) / 1e12,
                          "frac_of_sustained": step_flops / (ms_step / 1e3) / 1e12 / peaks["bf16_sustained"]},
        "phase_ms_per_step": per_step_ms,
        "peak_activation_gib": main_run["peak_bytes"] / 2**30,
        "workspace_gib": main_run["ws_bytes"] / 2**30,
        "chunk_buffers_gib": main_run["chunk_bytes"] / 2**30,
        "clocks": clocks,
        "memory_by_cp": memory_by_cp(upipe, S, Hq, Hkv, d, D, U, args.naive_kv),
    }
    if C > 1 and args.ring == 1:
        # all-to-all volume of one fwd+bwd step on this rank (the plan's per-stage buffers; each rank keeps
        # 1/C of every block), its event-timed duration on the comm stream, the bus bandwidth against
        # NVLink 5's 900 GB/s per direction, and the share of that time hidden behind compute
        off_rank = a2a_bytes(S_l, C, Hq, Hkv, d, U, args.naive_kv)["total"]
        comm_ms = per_step_ms.get("comm", 0.0)
        compute_ms = sum(v for k, v in per_step_ms.items() if k != "comm")
        result["a2a"] = {"bytes_per_step_off_rank": off_rank, "ms_per_step": comm_ms,
                         "bus_gbps": off_rank / (comm_ms / 1e3) / 1e9 if comm_ms > 0 else None, "peak_gbps": 900.0,
                         "overlap_fraction": min(1.0, max(0.0, (compute_ms + comm_ms - ms_step) / comm_ms))
                         if comm_ms > 0 else None,
                         "note": "comm-stream event time includes waiting for peers; overlap = share of it "
                                 "hidden behind the compute stream's kernels"}
    main_run["attn"].close()

    if not args.quick and not args.no_ulysses and U != Hq:
        try:
            ul = run(Hq, max(2, args.steps // 2), 1)
        except torch.OutOfMemoryError as exc:       # the max-context regime: Ulysses' full-head buffers do not fit
            main_run["attn"].close()
            torch.cuda.empty_cache()
            result["ulysses"] = {"chunk_heads": Hq, "oom": True, "error": str(exc).splitlines()[0][:200],
                                 "gpu_total_gib": torch.cuda.get_device_properties(dev).total_memory / 2**30}
            ul = None
    else:
        ul = None
    if ul is not None:
        ul_tok = S * max(2, args.steps // 2) / (ul["ms"] / 1e3) / world
        result["ulysses"] = {"chunk_heads": Hq, "value": ul_tok, "unit": "tokens/s/GPU",
                             "upipe_over_ulysses": tok_s / ul_tok,
                             "peak_activation_gib": ul["peak_bytes"] / 2**30,
                             "workspace_gib": ul["ws_bytes"] / 2**30,
                             "chunk_buffers_gib": ul["chunk_bytes"] / 2**30,
                             "activation_reduction": 1 - main_run["peak_bytes"] / ul["peak_bytes"],
                             "chunk_buffer_reduction": 1 - main_run["chunk_bytes"] / ul["chunk_bytes"],
                             "chunk_buffer_reduction_target": 1 - U / Hq}
        ul["attn"].close()

    if not args.quick and not args.no_e2e:
        # end to end through the public API: pinned host inputs -> HBM, fwd+bwd, dx -> pinned host
        # Every step copies its own x and dY from pinned host memory and reads its dx back, all inside
        # the timed region. The copies run on two copy streams (H2D, D2H) with double-buffered device
        # inputs, so step i+1's upload overlaps step i's backward, step i's y download overlaps its own backward
        # and its dx download step i+1's forward (the usual input pipeline of a training loop); nothing is
        # skipped or cached.
        attn = make_attn(U)
        xh = [x.cpu().pin_memory() for _ in range(2)]
        dyh = [dy.cpu().pin_memory() for _ in range(2)]
        dxh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
        yh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
        xd = [torch.empty_like(x) for _ in range(2)]
        dyd = [torch.empty_like(dy) for _ in range(2)]
        main_s = torch.cuda.current_stream()
        h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()                                   # noqa: E731
        bwd_done = [ev(), ev()]
        bwd_done[0].record(main_s)
        bwd_done[1].record(main_s)

        def e2e_step(i):
            b = i & 1
            with torch.cuda.stream(h2d):
                h2d.wait_event(bwd_done[b])                 # step i-2 no longer reads this input set
                xd[b].copy_(xh[b], non_blocking=True)
                x_ready = ev()
                x_ready.record(h2d)
                dyd[b].copy_(dyh[b], non_blocking=True)
                dy_ready = ev()
                dy_ready.record(h2d)
            main_s.wait_event(x_ready)
            y, saved = attn.forward(xd[b], *W, **NW)
            fwd_done = ev()
            fwd_done.record(main_s)
            with torch.cuda.stream(d2h):                    # y goes down while the backward runs
                d2h.wait_event(fwd_done)
                y.record_stream(d2h)
                yh[b].copy_(y, non_blocking=True)
            main_s.wait_event(dy_ready)
            dx, *_ = attn.backward(xd[b], *W, dyd[b], saved, **NW)
            bwd_done[b].record(main_s)
            with torch.cuda.stream(d2h):
                d2h.wait_event(bwd_done[b])
                dx.record_stream(d2h)
                dxh[b].copy_(dx, non_blocking=True)

        e2e_step(0)
        e2e_step(1)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ksteps = max(2, args.steps)                       # pipeline fill / drain amortised over the same K steps
        e0.record(main_s)
        h2d.wait_event(e0)
        for i in range(ksteps):
            e2e_step(i)
        main_s.wait_stream(d2h)                             # the last dx is on the host
        e1.record(main_s)
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1))
        result["e2e"] = {"value": S * ksteps / (ms / 1e3) / world, "unit": "tokens/s/GPU",
                         "h2d_bytes_per_step": 2 * x.numel() * 2, "d2h_bytes_per_step": 2 * x.numel() * 2,
                         "steps": ksteps, "api": "paper_2602_21196_b200.UPipeAttention.forward/backward",
                         "copies": "pinned host x, dY -> HBM and y, dx -> pinned host every step, on H2D/D2H copy "
                                   "streams overlapping the neighbouring steps' compute (double-buffered inputs); "
                                   "dW stays in HBM for the optimizer (per rank, bytes counted per rank)"}
        attn.close()

    if rank == 0 and world == 1 and not args.quick and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline()

    if pg is not None:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


if __name__ == "__main__":
    main()
