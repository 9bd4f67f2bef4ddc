"""Oracle: sparse attention forward/backward in float64 (test infrastructure only).

Restates:
  * full_attention           attention.py:95-109  (max-subtracted softmax of Q K^T / sqrt(d))
  * sparse attention         attention.py:153-187 (softmax renormalised over each query's
                             selected keys; uniform and ragged paths give the same math)
  * grouped attention        grouping.py:196-216  (members share the group's index set)
  * backward                 trainer.py:110-117   (autograd of gather -> einsum -> softmax ->
                             einsum: dQ per query; dK/dV summed over all queries selecting
                             a key), written analytically:
                                 dP = dO V_I^T,  dS = P * (dP - rowsum(dO * O)) * scale,
                                 dQ = dS K_I,  dK_I += dS^T Q,  dV_I += P^T dO.
LSE is returned in the natural log of the scaled logits.
"""

from __future__ import annotations

import numpy as np


def _softmax_rows(logits: np.ndarray) -> np.ndarray:
    z = logits - logits.max(axis=1, keepdims=True)
    w = np.exp(z)
    return w / w.sum(axis=1, keepdims=True)


def full_attention(q, k, v, scale=None):
    """attention.py:95-109."""
    q, k, v = (np.asarray(t, dtype=np.float64) for t in (q, k, v))
    scale = 1.0 / np.sqrt(q.shape[1]) if scale is None else scale
    return _softmax_rows(q @ k.T * scale) @ v


def grouped_attention_fwd(q, k, v, members, group_sets, scale=None):
    """One head: members[g] = query rows of group g, group_sets[g] = its key ids.

    Returns (out [Lq, d], lse [Lq]) in float64.
    """
    q, k, v = (np.asarray(t, dtype=np.float64) for t in (q, k, v))
    scale = 1.0 / np.sqrt(q.shape[1]) if scale is None else scale
    out = np.zeros((q.shape[0], v.shape[1]))
    lse = np.zeros(q.shape[0])
    for mem, sel in zip(members, group_sets):
        mem = np.asarray(mem, dtype=np.int64)
        sel = np.asarray(sel, dtype=np.int64)
        if sel.size == 0:
            raise ValueError("every query needs at least one selected index")
        logits = q[mem] @ k[sel].T * scale
        mx = logits.max(axis=1, keepdims=True)
        w = np.exp(logits - mx)
        ssum = w.sum(axis=1, keepdims=True)
        out[mem] = (w / ssum) @ v[sel]
        lse[mem] = (mx + np.log(ssum))[:, 0]
    return out, lse


def grouped_attention_bwd(q, k, v, members, group_sets, dout, scale=None):
    """Analytic gradients of grouped_attention_fwd (trainer.py:110-117 autograd)."""
    q, k, v, dout = (np.asarray(t, dtype=np.float64) for t in (q, k, v, dout))
    scale = 1.0 / np.sqrt(q.shape[1]) if scale is None else scale
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for mem, sel in zip(members, group_sets):
        mem = np.asarray(mem, dtype=np.int64)
        sel = np.asarray(sel, dtype=np.int64)
        p = _softmax_rows(q[mem] @ k[sel].T * scale)
        o = p @ v[sel]
        do = dout[mem]
        dp = do @ v[sel].T
        ds = p * (dp - (do * o).sum(axis=1, keepdims=True)) * scale
        dq[mem] = ds @ k[sel]
        if sel.size < 2 or np.all(np.diff(sel) > 0):   # unique keys: plain fancy-index add
            dk[sel] += ds.T @ q[mem]
            dv[sel] += p.T @ do
        else:
            np.add.at(dk, sel, ds.T @ q[mem])
            np.add.at(dv, sel, p.T @ do)
    return dq, dk, dv


def rows_attention_fwd(q, k, v, index_lists, scale=None):
    """Per-query (ragged) sets: attention.py:176-183."""
    members = [[i] for i in range(len(index_lists))]
    return grouped_attention_fwd(q, k, v, members, index_lists, scale)


def rows_attention_bwd(q, k, v, index_lists, dout, scale=None):
    members = [[i] for i in range(len(index_lists))]
    return grouped_attention_bwd(q, k, v, members, index_lists, dout, scale)
