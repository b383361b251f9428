"""Helpers for the GPU parity tests: numpy (oracle side) <-> torch CUDA (libcp side)."""
import numpy as np
import torch


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def dev_tensor(Z):
    return torch.from_numpy(np.ascontiguousarray(Z, dtype=np.float64)).cuda()


def dev_factor(A):
    """numpy I x R -> CUDA float64 tensor (I x R) stored column-major."""
    A = np.asarray(A, dtype=np.float64)
    t = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # (R, I) contiguous
    return t.t()


def host_factor(t):
    return np.asfortranarray(t.detach().cpu().numpy())


def host_tensor(t):
    return t.detach().cpu().numpy()
