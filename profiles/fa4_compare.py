"""Library comparison (context only, not part of the product path): FlashAttention-4 (the CuTe-DSL sm_100 kernels
vendored in vllm's `vllm_flash_attn.cute`) forward and backward at the attention shapes of the bench, and ours
through the C ABI on the same inputs in the same process, both timed the same way (CUDA events, median of `reps`
launches after a warm-up; `--ours` adds our lines). FLOP convention as in DESIGN §7: causal fwd 4·d·S(S+1)/2 per
head, bwd 10·d·S(S+1)/2 per head. The FA4 backward time includes its preprocess (row-dot) and postprocess (dQ
conversion) kernels; ours is the main kernel alone (the row-dot is fused in our dO GEMM, the conversion is a separate
~0.2 ms launch).

usage: python profiles/fa4_compare.py [--two-cta both|on|off] [--ours] S:nq:nkv ...
"""
import argparse
import json
import os
import sys

import torch


class ClockSampler:
    """nvidia-smi-equivalent SM clock / power samples (NVML) taken every 5 ms while a timed region runs."""

    def __init__(self):
        import threading
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.on = False
        self.samples = []
        self.threading = threading

    def __enter__(self):
        self.samples = []
        self.on = True

        def loop():
            import time
            while self.on:
                self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                     self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
                time.sleep(0.005)
        self.t = self.threading.Thread(target=loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self.on = False
        self.t.join()

    def summary(self):
        if not self.samples:
            return None
        cl = sorted(c for c, _ in self.samples)
        pw = sorted(p for _, p in self.samples)
        return {"sm_mhz_median": cl[len(cl) // 2], "power_w_median": round(pw[len(pw) // 2], 1), "n": len(cl)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shapes", nargs="*", default=["131072:8:2"])
    ap.add_argument("--two-cta", default="both")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ours", action="store_true")
    args = ap.parse_args()
    from vllm.vllm_flash_attn.cute import interface as fa, utils as fau

    modes = {"both": [False, True], "on": [True], "off": [False]}[args.two_cta]
    for shp in args.shapes:
        S, nq, nkv = (int(v) for v in shp.split(":"))
        d = 128
        g = torch.Generator(device="cuda").manual_seed(0)
        q = torch.randn(1, S, nq, d, device="cuda", dtype=torch.bfloat16, generator=g)
        k = torch.randn(1, S, nkv, d, device="cuda", dtype=torch.bfloat16, generator=g)
        v = torch.randn(1, S, nkv, d, device="cuda", dtype=torch.bfloat16, generator=g)
        do = torch.randn(1, S, nq, d, device="cuda", dtype=torch.bfloat16, generator=g)
        fl = d * S * (S + 1) / 2 * nq
        for two in modes:
            fau._fa_disable_2cta_cuda12 = not two
            fau._fa_disable_2cta_enabled = not two
            try:
                qq, kk, vv = (t.detach().clone().requires_grad_(True) for t in (q, k, v))
                out = fa.flash_attn_func(qq, kk, vv, causal=True)
                out = out[0] if isinstance(out, tuple) else out
                out.backward(do)                      # compile both directions
                torch.cuda.synchronize()
                fwd, bwd = [], []
                cs = ClockSampler()
                cs.__enter__()
                for _ in range(args.reps):
                    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                    qq.grad = kk.grad = vv.grad = None
                    e0.record()
                    out = fa.flash_attn_func(qq, kk, vv, causal=True)
                    out = out[0] if isinstance(out, tuple) else out
                    e1.record()
                    out.backward(do)
                    e2.record()
                    torch.cuda.synchronize()
                    fwd.append(e0.elapsed_time(e1))
                    bwd.append(e1.elapsed_time(e2))
                cs.__exit__()
                cf = ClockSampler()                       # forward alone (no autograd), for its clock
                with torch.no_grad(), cf:
                    for _ in range(args.reps):
                        fa.flash_attn_func(q, k, v, causal=True)
                    torch.cuda.synchronize()
                f, b = sorted(fwd)[len(fwd) // 2], sorted(bwd)[len(bwd) // 2]
                print(json.dumps({"impl": "fa4", "two_cta": two, "S": S, "nq": nq, "nkv": nkv, "d": d,
                                  "fwd_ms": f, "fwd_tflops": 4 * fl / f / 1e9, "bwd_ms": b,
                                  "bwd_tflops": 10 * fl / b / 1e9,
                                  "clocks": {"fwd": cf.summary(), "fwd_bwd": cs.summary()}}), flush=True)
            except Exception as ex:  # noqa: BLE001 - a library failure is reported, not fatal
                print(json.dumps({"impl": "fa4", "two_cta": two, "S": S, "error": repr(ex)[:400]}), flush=True)
            torch.cuda.empty_cache()
        if args.ours:
            sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            from paper_2602_21196_b200 import upipe
            # our layout: [S][heads][d] rows (the same memory as FA4's [1][S][heads][d])
            qq, kk, vv, dd = (t[0].contiguous() for t in (q, k, v, do))
            o = torch.empty((S, nq, d), dtype=torch.bfloat16, device="cuda")
            lse = torch.empty((nq, S), dtype=torch.float32, device="cuda")
            delta = torch.empty((S, nq), dtype=torch.float32, device="cuda")
            dq = torch.zeros((nq * d, S), dtype=torch.float32, device="cuda")   # dim-major, as the layer uses it
            dk = torch.empty((S, nkv, d), dtype=torch.float32, device="cuda")
            dv = torch.empty((S, nkv, d), dtype=torch.float32, device="cuda")

            def fwd_o():
                upipe.upipe_attn_core_fwd(qq, kk, vv, o, lse, S, nq, nkv, d, 1, nq * d, nkv * d, nq * d, S)

            def bwd_o():
                upipe.upipe_attn_core_bwd(qq, kk, vv, dd, lse, delta, dq, dk, dv, S, nq, nkv, d, 1, nq * d, nkv * d,
                                          nq * d, S, nq, dq_dim_major=True)

            fwd_o()
            upipe.upipe_rowdot(dd, nq * d, o, nq * d, delta, nq, S, nq, d)
            fwd, bwd = [], []
            clk = {}
            for f_, acc, nm in ((fwd_o, fwd, "fwd"), (bwd_o, bwd, "bwd")):
                f_()
                cs = ClockSampler()
                cs.__enter__()
                for _ in range(args.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    f_()
                    e1.record()
                    torch.cuda.synchronize()
                    acc.append(e0.elapsed_time(e1))
                cs.__exit__()
                clk[nm] = cs.summary()
            f, b = sorted(fwd)[len(fwd) // 2], sorted(bwd)[len(bwd) // 2]
            print(json.dumps({"impl": "ours", "S": S, "nq": nq, "nkv": nkv, "d": d, "fwd_ms": f,
                              "fwd_tflops": 4 * fl / f / 1e9, "bwd_ms": b, "bwd_tflops": 10 * fl / b / 1e9,
                              "clocks": clk}), flush=True)
            del qq, kk, vv, dd, o, lse, delta, dq, dk, dv
            torch.cuda.empty_cache()


if __name__ == "__main__":
    sys.exit(main())
