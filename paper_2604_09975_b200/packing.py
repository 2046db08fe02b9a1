"""Client-side slot layouts of EncFormer (plain numpy data arrangement, no CKKS arithmetic).

These are the layouts the CKKS kernels consume and produce (SCP):
  segment-column, folded-diagonal, head-major,
  the score-friendly column permutation pi_S and the G8 padding of Q/K blocks.
Written independently of oracle/kernels.py (the two share no code).
"""
import numpy as np


def seg_columns(X, m, C, group, n):
    """Slot vector whose segment c < C holds column X[:, group*C + c] (zero beyond X's columns)."""
    out = np.zeros(n, dtype=np.complex128)
    cols = X[:, group * C:(group + 1) * C]
    k = cols.shape[1]
    out[:k * m] = cols.T.reshape(-1)
    return out


def complexified_inputs(X, m, C, n):
    """x~_u = x^(2u) + i x^(2u+1), u < ceil(G/2)."""
    G = -(-X.shape[1] // C)
    return [seg_columns(X, m, C, 2 * u, n) + 1j * seg_columns(X, m, C, 2 * u + 1, n) for u in range((G + 1) // 2)]


def unpack_columns(z, m, C, ncols):
    """Inverse of seg_columns for one output block: first ncols segments -> (m, ncols)."""
    return np.asarray(z[:ncols * m]).reshape(ncols, m).T


def score_perm(H, d_h):
    """Column order pi_S(h, u) = u H + h: returns idx with Wpi[:, j] = W[:, idx[j]]."""
    idx = np.empty(H * d_h, dtype=np.int64)
    for u in range(d_h):
        for h in range(H):
            idx[u * H + h] = h * d_h + u
    return idx


def qkv_weight(WQ, WK, WV, H, d_h, C, C_qk):
    """Pre-permuted, padded QKV weight (App. A.2 + G8): Q and K blocks hold C_qk used columns of
    W^{pi_S} followed by C - C_qk zero columns; V blocks are head-major (pi_V = identity)."""
    d = WQ.shape[0]
    perm = score_perm(H, d_h)
    nqk = -(-(H * d_h) // C_qk)
    nv = -(-(H * d_h) // C)
    W = np.zeros((d, (2 * nqk + nv) * C))
    for i, Wm in enumerate((WQ[:, perm], WK[:, perm])):
        for b in range(nqk):
            blk = Wm[:, b * C_qk:(b + 1) * C_qk]
            W[:, (i * nqk + b) * C:(i * nqk + b) * C + blk.shape[1]] = blk
    W[:, 2 * nqk * C:2 * nqk * C + WV.shape[1]] = WV
    return W, nqk, nv


def folded_diag_blocks(Ph, m, H_blk, stride, n):
    """P_fd blocks: segment h~ stride + t holds p_t + i p_{t+m/2} of local head h~,
    p_t[j] = P[j, (j+t) mod m]."""
    H = Ph.shape[0]
    j = np.arange(m)
    blocks = []
    for l in range(-(-H // H_blk)):
        z = np.zeros(n, dtype=np.complex128)
        for hh in range(H_blk):
            h = l * H_blk + hh
            if h >= H:
                break
            for t in range(m // 2):
                s = hh * stride + t
                z[s * m:(s + 1) * m] = Ph[h][j, (j + t) % m] + 1j * Ph[h][j, (j + t + m // 2) % m]
        blocks.append(z)
    return blocks


def k_min(n_entries, n):
    return -(-int(n_entries) // (2 * int(n)))
