"""Closed-form eigenpairs used as parity pins (test infrastructure; neither the oracle nor the
CUDA path).  SURVEY 8(c.4): the 3-D 7-point Dirichlet Laplacian (center 6, neighbours -1, rows
x + N(y + N z)) is diagonalised by the sine tensor basis
    v_{k1,k2,k3}(x, y, z) = s_{k1}(x) s_{k2}(y) s_{k3}(z),  s_k(i) = sqrt(2/(N+1)) sin(k pi (i+1)/(N+1)),
    lambda = sum_d (2 - 2 cos(k_d pi / (N+1))),  k_d = 1..N.
C3 (128^3, d = 0) has exactly degenerate clusters; each cluster's eigenspace is spanned by the
index permutations of one (k1, k2, k3)."""
import itertools

import numpy as np


def laplace3d_lowest(N, p, kmax=8):
    """The p smallest eigenvalues (ascending; p must end on a cluster boundary) with orthonormal
    eigenvectors (n x p) and the cluster groups (lists of column indices)."""
    c = 2.0 - 2.0 * np.cos(np.arange(1, kmax + 1) * np.pi / (N + 1))
    trip = sorted(itertools.product(range(kmax), repeat=3), key=lambda t: (c[t[0]] + c[t[1]] + c[t[2]], t))
    lam = np.array([c[a] + c[b] + c[d] for a, b, d in trip])
    if p < len(lam):
        assert lam[p] - lam[p - 1] > 1e-12 * lam[p], "p splits a cluster"
    i = np.arange(N)
    S = np.sqrt(2.0 / (N + 1)) * np.sin(np.outer(i + 1, np.arange(1, kmax + 1)) * np.pi / (N + 1))  # N x kmax
    V = np.empty((N ** 3, p))
    for col, (a, b, d) in enumerate(trip[:p]):
        V[:, col] = np.einsum("z,y,x->zyx", S[:, d], S[:, b], S[:, a]).ravel()  # x fastest
    groups, cur = [], [0]
    for j in range(1, p):
        if abs(lam[j] - lam[j - 1]) <= 1e-12 * lam[j]:
            cur.append(j)
        else:
            groups.append(cur)
            cur = [j]
    groups.append(cur)
    return lam[:p], V, groups


def sin_angle(X, V):
    """Largest principal angle (its sine) between span(X) and span(V), both orthonormal columns:
    || X - V (V^T X) ||_2."""
    R = X - V @ (V.T @ X)
    return float(np.linalg.norm(R, 2))
