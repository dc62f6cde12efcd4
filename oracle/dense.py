"""Tall-skinny Grassmann steps of the oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Textbook linear algebra with numpy library primitives:
  * projection onto the horizontal space at U:  P_U(G) = G - U (U^T G)   (
    Grassmann geometry of PAPER.md:70-71,120, Edelman99)
  * QR retraction:  Q factor of the thin QR of U + xi, with signs fixed so that R_ii > 0
    (SPEC.md:324-332).  LAPACK Householder QR (numpy.linalg.qr) + sign flip.
"""
from __future__ import annotations

import numpy as np


def project(U: np.ndarray, G: np.ndarray) -> np.ndarray:
    U = np.asarray(U, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    M = U.T @ G
    return G - U @ M


def retract(U: np.ndarray, xi: np.ndarray):
    """Returns (Q, R) with Q R = U + xi, R upper triangular, diag(R) > 0."""
    Y = np.asarray(U, dtype=np.float64) + np.asarray(xi, dtype=np.float64)
    Q, R = np.linalg.qr(Y, mode="reduced")
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return Q * s[None, :], R * s[:, None]


def dot(x: np.ndarray, y: np.ndarray) -> float:
    """<x, y> = sum_{i,l} x_il y_il (Euclidean metric on the horizontal space)."""
    return float(np.sum(np.asarray(x, dtype=np.float64) * np.asarray(y, dtype=np.float64)))
