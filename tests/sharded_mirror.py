"""Test infrastructure: a numpy restatement of the column-sharded decomposition
that csrc/sharded.inc implements, run on CPU ranks of a
torch.distributed gloo group.  It uses the same shard ranges
(cnmf_shard_begin), the same split of work (replicated A half, local B half,
one B-check all-reduce per iteration, sketch products summed across ranks,
CholeskyQR2 with all-reduced Grams for row-sharded bases) and checks it
against the single-process oracle.  Only tests import this module.
"""
import numpy as np
import torch
import torch.distributed as dist

KDEAD = 1e-12  # solvers.cpp:19


def allreduce(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def shard(n, rank, world):
    return n * rank // world, n * (rank + 1) // world


def cholqr2_rows(y_local):
    """Orthonormal basis of a row-sharded matrix: two CholeskyQR passes with
    the l x l Gram summed over ranks (launch_thin_qr_dist)."""
    q = y_local
    for _ in range(2):
        g = allreduce(q.T @ q)
        r = np.linalg.cholesky(g).T
        q = q @ np.linalg.inv(r)
    return q


def householder_q(y):
    """Thin Q of a replicated matrix (the single-GPU path's role; any
    orthonormal basis of the span serves, only spans matter)."""
    return np.linalg.qr(y)[0]


def range_finder_sharded(x_local, q, w, omega, transpose, lo, hi):
    """range_finder_impl (compression.cpp:23-42) on the column shard
    x_local = X[:, lo:hi].  transpose=False: replicated basis of range(X)
    (omega is the full n x q sketch); True: this rank's rows of a basis of
    range(X^T) (omega is the d x q sketch)."""
    nn = lambda s_local: allreduce(x_local @ s_local)  # X S, summed over ranks
    tn = lambda t: x_local.T @ t                      # local rows of X^T T
    if not transpose:
        basis = householder_q(nn(omega[lo:hi]))
        for _ in range(w):
            z = cholqr2_rows(tn(basis))
            basis = householder_q(nn(z))
    else:
        basis = cholqr2_rows(tn(omega))
        for _ in range(w):
            z = householder_q(nn(basis))
            basis = cholqr2_rows(tn(z))
    return basis


def fasthals_rp_steps_sharded(xhat_local, xcheck, a, b_local, ahat, bchk, left, right_local,
                              steps, normalize_a=True):
    """fasthals_rp_step (solvers.cpp:414-456) with the A half replicated and the
    B half on this rank's rows; B-check = sum_g R_g B_g all-reduced each step.
    Dead / emptied components are not expected in the test data (asserted)."""
    a = a.copy()
    b = b_local.copy()
    k = a.shape[1]
    for _ in range(steps):
        h = xcheck @ bchk                      # 421
        g = bchk.T @ bchk                      # 422
        for j in range(k):                     # 423-437
            assert g[j, j] >= KDEAD
            v = a[:, j] + (h[:, j] - a @ g[:, j]) / g[j, j]
            a[:, j] = np.maximum(v, 0.0)
            nrm = np.linalg.norm(a[:, j])
            assert nrm > 0.0
            if normalize_a:
                a[:, j] /= nrm
        ahat = left.T @ a                      # 438
        p = xhat_local.T @ ahat                # 442 (local rows)
        w = ahat.T @ ahat                      # 443 (replicated)
        nonzero = np.zeros(k)
        for j in range(k):                     # 444-453
            assert w[j, j] >= KDEAD
            v = b[:, j] + (p[:, j] - b @ w[:, j]) / w[j, j]  # 480-490 (alpha = beta = 0)
            b[:, j] = np.maximum(v, 0.0)
            nonzero[j] = float(np.any(b[:, j] != 0.0))
        red = allreduce(np.concatenate([(right_local.T @ b).ravel(), nonzero]))  # 454 + flags
        bchk = red[: bchk.size].reshape(bchk.shape)
        assert np.all(red[bchk.size:] > 0.0)   # no globally emptied column
    return a, b, ahat, bchk
