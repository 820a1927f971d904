"""Helpers shared by the GPU parity tests (tests/ only)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def dev(a):
    """numpy (fp64) -> CUDA float32 tensor."""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().double().cpu().numpy()


def r32(a):
    """Round to fp32 (the GPU's storage type); the oracle then runs fp64 on these."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def maxrel(a, b):
    """max|a - b| / max|b| (SURVEY.md 8(d) gradient metric)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (den if den > 0 else 1.0))


def l2rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
