"""Boundary-weighted L1 loss, Eq. 2 of the paper:

    L_Total = (1 - lambda) L1(X_Uniform, Y_Uniform) + lambda L1(X_Bound, Y_Bound)

L1 = mean absolute error per term, pooled over samples and channels
for vector fields (D = 3: mean over the n x D residuals, as S:L78 pools the
MSE; R28); an empty boundary set makes the
effective lambda' = 0 (R11); subgradient sgn(0) = 0 (R11).
"""
import numpy as np


def loss_and_grad(y_u, t_u, y_b, t_b, lam):
    """Returns (total, l1_uniform, l1_boundary, dy_u, dy_b) in float64; y, t of
    shape (n,) or (n, D) (dy flattened in the same element order)."""
    y_u = np.asarray(y_u, np.float64).reshape(-1)
    t_u = np.asarray(t_u, np.float64).reshape(-1)
    y_b = np.asarray(y_b, np.float64).reshape(-1)
    t_b = np.asarray(t_b, np.float64).reshape(-1)
    lam_eff = float(lam) if y_b.size > 0 else 0.0
    l1_u = float(np.mean(np.abs(y_u - t_u))) if y_u.size else 0.0
    l1_b = float(np.mean(np.abs(y_b - t_b))) if y_b.size else 0.0
    total = (1.0 - lam_eff) * l1_u + lam_eff * l1_b
    dy_u = (1.0 - lam_eff) * np.sign(y_u - t_u) / max(y_u.size, 1)
    dy_b = lam_eff * np.sign(y_b - t_b) / max(y_b.size, 1)
    return total, l1_u, l1_b, dy_u, dy_b
