"""CPU checks of bench.py's algorithmic byte/flop counts (the roofline numerators).

The per-node byte counts follow from the data layout alone (fp64, nx = 4, ny = 2, K = 32 nodes
per run): they are restated here from DESIGN.md's table rather than from bench.py's formulas.
"""
import numpy as np

import bench

WIENER_A = np.array([[1, 0, 1, 0], [0, 1, 0, 1], [0, 0, 1, 0], [0, 0, 0, 1]], bool)  # I - dt F
WIENER_U = np.array([[0, 0], [0, 0], [1, 0], [0, 1]], bool)  # sqrt(dt) L chol(W)


def test_canonical_solve_bytes():
    # y (2 doubles) read once, (S, v) (10 + 4 doubles) written and read once, x (4) written:
    # 8 * (2 + 2 * 14 + 4) = 272 B/node
    c = bench.alg_counts(4, 2)
    assert c["solve"][1] == 272


def test_lowrank_record_bytes():
    # R-P2REC: record [S U | U^T v] = 2 * 5 doubles = 80 B instead of (S, v) = 112 B
    dense = bench.alg_counts(4, 2)
    lr = bench.alg_counts(4, 2, nw=2, zero_b=True)
    assert dense["k_p1_down"][1] - lr["k_p1_down"][1] == 8 * (14 - 10)
    assert dense["k_p2_down"][1] - lr["k_p2_down"][1] == 8 * (14 - 10)


def test_compact_record_bytes_and_flops():
    # R-P2REC-C: S[:, 2:4] (7 distinct values) + v[2:4] = 9 doubles = 72 B; pass 2 forms S U and
    # U^T v (10 products = 5 FMA-equivalents) that the 80 B record carried
    lr = bench.alg_counts(4, 2, nw=2, zero_b=True, amask=WIENER_A, umask=WIENER_U)
    um = np.ones((4, 2), bool)
    lr_dense_u = bench.alg_counts(4, 2, nw=2, zero_b=True, amask=WIENER_A, umask=um)
    assert lr_dense_u["k_p1_down"][1] - lr["k_p1_down"][1] == 8
    assert lr_dense_u["k_p2_down"][1] - lr["k_p2_down"][1] == 8
    assert lr["k_p1_down"][1] == 104
    # the compact pass-2 step = the 80 B-record step on the same masks + 5 FMAs
    nA, nU = int(WIENER_A.sum()), int(WIENER_U.sum())
    r, N = 2, 4
    chol = sum((a + 1) * int(WIENER_U[:, a].sum()) for a in range(r)) + r * (r - 1) // 2 * (r + 1) + r
    assert lr["k_p2_down"][0] == 2 * (nA + nU + chol + r * N + r * r + nU + 5)


def test_lowrank_transition_flops_without_masks():
    # the low-rank pass-2 step replaces the dense (I + C S)^-1 A solve whenever the record is the
    # low-rank one, masks or not (regression: it must not fall back to the dense count)
    dense = bench.alg_counts(4, 2)
    lr = bench.alg_counts(4, 2, nw=2, zero_b=True)
    assert lr["k_p2_down"][0] < dense["k_p2_down"][0]
