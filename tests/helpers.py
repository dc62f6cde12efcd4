"""Shared test helpers (comparison metric of DESIGN.md §4 / SURVEY.md §8(c) reading #15)."""
import numpy as np

TOL = 1e-9  # north star: max relative error 1e-9 on F, grad and Hv (fp64)


def colwise_relerr(x, ref):
    """max over columns l of max_i |x_il - ref_il| / max_i |ref_il|  (normwise-inf per column)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if x.ndim == 1:
        x, ref = x[:, None], ref[:, None]
    den = np.max(np.abs(ref), axis=0)
    den[den == 0] = 1.0
    return float(np.max(np.max(np.abs(x - ref), axis=0) / den))


def scalar_relerr(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.maximum(np.abs(ref), 1e-300)
    return float(np.max(np.abs(x - ref) / den))


def to_np(t):
    return t.detach().cpu().numpy()
