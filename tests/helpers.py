"""Shared test helpers (no method arithmetic here)."""
import numpy as np
import torch

import synth
from paper_1703_09268_b200 import api


def grid_of(p):
    return api.Grid.of(p)


def to_dev(a: np.ndarray, dtype=torch.complex128) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().astype(np.complex128)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def random_fields(n_ext, nrhs, seed=1):
    return synth.random_complex((nrhs, n_ext), seed)
