"""Oracle: predictor training step (test infrastructure only; see oracle/__init__.py).

Restates pkg/src/dynsparse/predictor.py:
  * cos_terms        predictor.py:103-124  per-row cosine loss and its gradient
  * norm_terms       predictor.py:127-136  relative Frobenius loss and its gradient
  * loss_and_grads   predictor.py:151-194  A_hat = (X_r W_q)(X W_k)^T, G = dL/dA_hat,
                                           dW_q = X_r^T (G K_lr), dW_k = X^T (G^T Q_lr)
  * adam / train     predictor.py:197-214  Adam with bias correction; non-finite
                                           gradients skip the update
"""

from __future__ import annotations

import numpy as np

COS_WEIGHT, NORM_WEIGHT, NORM_FLOOR = 0.95, 0.05, 1e-12


def cos_terms(a_hat, target):
    n = a_hat.shape[0]
    a_norm = np.linalg.norm(a_hat, axis=1)
    t_norm = np.linalg.norm(target, axis=1)
    live = t_norm > NORM_FLOOR
    cos = np.zeros(n)
    grad = np.zeros_like(a_hat)
    nz = live & (a_norm > NORM_FLOOR)
    if np.any(nz):
        an, tn = a_norm[nz, None], t_norm[nz, None]
        dots = np.sum(a_hat[nz] * target[nz], axis=1, keepdims=True)
        c = dots / (an * tn)
        cos[nz] = c[:, 0]
        grad[nz] = -(target[nz] / (an * tn) - c * a_hat[nz] / an**2) / n
    return float(np.sum(np.where(live, 1.0 - cos, 0.0)) / n), grad


def norm_terms(a_hat, target):
    denom = max(float(np.linalg.norm(target)), NORM_FLOOR)
    diff = a_hat - target
    dist = float(np.linalg.norm(diff))
    grad = diff / (denom * dist) if dist > NORM_FLOOR else np.zeros_like(a_hat)
    return dist / denom, grad


def loss_and_grads(w_q, w_k, x, target, rows=None):
    """-> (cos_loss, norm_loss, total, grad_wq, grad_wk)."""
    x = np.asarray(x, dtype=np.float64)
    xr = x if rows is None else x[np.asarray(rows, dtype=np.int64)]
    q_lr, k_lr = xr @ w_q, x @ w_k
    a_hat = q_lr @ k_lr.T
    target = np.asarray(target, dtype=np.float64)
    cl, gc = cos_terms(a_hat, target)
    nl, gn = norm_terms(a_hat, target)
    g = COS_WEIGHT * gc + NORM_WEIGHT * gn
    return cl, nl, COS_WEIGHT * cl + NORM_WEIGHT * nl, xr.T @ (g @ k_lr), x.T @ (g.T @ q_lr)


def adam(w, grad, m, v, lr, b1, b2, eps, step):
    m *= b1
    m += (1.0 - b1) * grad
    v *= b2
    v += (1.0 - b2) * grad**2
    w -= lr * (m / (1.0 - b1**step)) / (np.sqrt(v / (1.0 - b2**step)) + eps)


def train(w_q, w_k, x, target, steps, lr=1e-3, rows=None, b1=0.9, b2=0.999, eps=1e-8):
    """`steps` train_step calls from zero Adam state -> (w_q, w_k, loss history)."""
    w_q, w_k = np.array(w_q, dtype=np.float64), np.array(w_k, dtype=np.float64)
    mq, vq, mk, vk = (np.zeros_like(w_q) for _ in range(4))
    hist, step = [], 0
    for _ in range(steps):
        _, _, tot, gq, gk = loss_and_grads(w_q, w_k, x, target, rows)
        if np.all(np.isfinite(gq)) and np.all(np.isfinite(gk)):
            step += 1
            adam(w_q, gq, mq, vq, lr, b1, b2, eps, step)
            adam(w_k, gk, mk, vk, lr, b1, b2, eps, step)
        hist.append(tot)
    return w_q, w_k, np.array(hist)
