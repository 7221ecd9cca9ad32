"""Helpers shared by the -m gpu tests (no method arithmetic here)."""
import numpy as np
import torch


def dev():
    if not torch.cuda.is_available():
        raise RuntimeError("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)


def to_bf16(a: np.ndarray) -> torch.Tensor:
    """fp64 array of exactly-representable bf16 values -> cuda bf16 tensor (bit exact)."""
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16)
    assert torch.equal(t.to(torch.float64), torch.from_numpy(np.asarray(a, dtype=np.float64))), "not bf16-exact"
    return t.to(dev())


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def errs(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    return rel, float(np.abs(got - want).max())


# Every assert_close records its achieved errors; tests/conftest.py writes them to
# $UPIPE_PARITY_REPORT (JSON) at the end of the session (the committed profiles/parity_r02.json).
RECORDS = []


def assert_close(name, got, want, rel_tol, abs_tol):
    import os
    rel, mx = errs(got, want)
    RECORDS.append({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "tensor": name,
                    "rel_l2": float(rel), "max_abs": mx, "rel_tol": rel_tol, "abs_tol": abs_tol,
                    "ok": bool(np.isfinite(rel) and rel <= rel_tol and mx <= abs_tol)})
    assert np.isfinite(rel) and rel <= rel_tol and mx <= abs_tol, f"{name}: rel L2 {rel:.3e} (tol {rel_tol}), max|d| {mx:.3e} (tol {abs_tol})"
    return rel, mx
