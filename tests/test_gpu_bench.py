"""The bench.py contract (one JSON line with the keys the driver reads), run on a small sequence."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--seq", "8192", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "clocks", "e2e", "ulysses"):
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 3 and j["warmup"] == 3 and j["value"] > 0
    assert j["gpu_launches"] > 0                                   # our kernels ran in the timed region
    rf = j["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1.2
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "workload" in j["config"]
    assert j["ulysses"]["chunk_buffer_reduction"] == pytest.approx(1 - 8 / 32)


def test_bench_reference_arm_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    j = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert j["impl"] == "reference" and j["value"] > 0 and j["cpu_baseline"]["kind"] == "oracle"
    assert j["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.timeout(900)
@pytest.mark.parametrize("direct", [False, True])
def test_bench_multi_rank_path_on_one_gpu(direct):
    # the N > 1 path of bench.py (torchrun launch, IPC transport, max-over-ranks timing, the a2a and memory_by_cp
    # keys) with both ranks on cuda:0 (UPIPE_BENCH_SAME_GPU=1, gloo group): the contract line, not a timing
    import json
    import os
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--seq", "8192", "--transport", "ipc", "--no-ulysses", "--no-e2e"]
    if direct:
        cmd.append("--direct")
    r = subprocess.run(cmd, env=dict(os.environ, UPIPE_BENCH_SAME_GPU="1", UPIPE_QUIET="1"), capture_output=True,
                       text=True, timeout=800)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["unit"] == "tokens/s/GPU"
    assert abs(d["tokens_per_s_total"] / d["value"] - 2) < 1e-6
    assert d["config"]["transport"] == ("ipc-direct" if direct else "ipc")
    assert d["a2a"]["bytes_per_step_off_rank"] > 0 and d["gpu_launches"] > 0
    assert set(d["memory_by_cp"]) >= {"1", "2", "4", "8"}
