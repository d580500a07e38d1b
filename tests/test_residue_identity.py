"""The identity behind the residue-plane path of the fused per-vertex relight,
checked in exact arithmetic on the paper's bottom-up recursion (-m "not gpu", no GPU code):

    BU^k(roll(F, Q)) = roll(BU^k(roll(F, Q mod 2^k)), Q div 2^k)

for the X, Y and Z fields' filters (h_s = [1,1], h_t = [1,2,1], decimated by 2), every
Q on a small periodic grid, and the box-projection shift as the weighted sum of four such rolls.
Integer-valued fields and float64 sums of small integers are exact, so the comparison is ==."""
import numpy as np
import pytest


def bu(F, kind):
    """one bottom-up level of a periodic field: X: [1,1] along rows, [1,2,1] along columns; Y the
    transpose; Z [1,2,1] both (times 4, to stay in integers)"""
    def hs(A, ax):
        return A + np.roll(A, -1, axis=ax)

    def ht(A, ax):
        return A + 2 * np.roll(A, -1, axis=ax) + np.roll(A, -2, axis=ax)
    if kind == "X":
        G = ht(hs(F, 0), 1)
    elif kind == "Y":
        G = hs(ht(F, 0), 1)
    else:
        G = ht(ht(F, 0), 1)
    return G[0::2, 0::2]


def roll(F, q):
    return np.roll(F, shift=(q[0], q[1]), axis=(0, 1))   # roll(F, q)(y, x) = F(y - qy, x - qx)


@pytest.mark.parametrize("kind", ["X", "Y", "Z"])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_bottom_up_commutes_with_rolls_by_residues(kind, k):
    rng = np.random.default_rng(7 + k)
    N = 16
    F = rng.integers(-50, 50, size=(N, N)).astype(np.float64)
    for Qy in range(0, N, 3):
        for Qx in range(0, N, 5):
            lhs = roll(F, (Qy, Qx))
            rhs = roll(F, (Qy % 2 ** k, Qx % 2 ** k))
            for _ in range(k):
                lhs = bu(lhs, kind)
                rhs = bu(rhs, kind)
            rhs = roll(rhs, (Qy // 2 ** k, Qx // 2 ** k))
            assert np.array_equal(lhs, rhs)


def test_box_shift_is_four_rolls_and_the_planes_reproduce_it():
    """S F = sum_ab w_ab roll(F, q + (a, b)); its k-level bottom-up equals the weighted sum of the
    rolled residue planes -- the per-vertex formula of the fused path"""
    rng = np.random.default_rng(3)
    N, k = 16, 2
    F = rng.integers(-50, 50, size=(N, N)).astype(np.float64)
    wy1, wx1 = 0.25, 0.75                                   # dyadic weights: exact in float64
    w = {(0, 0): (1 - wy1) * (1 - wx1), (0, 1): (1 - wy1) * wx1, (1, 0): wy1 * (1 - wx1), (1, 1): wy1 * wx1}
    planes = {}
    for ry in range(2 ** k):
        for rx in range(2 ** k):
            P = roll(F, (ry, rx))
            for _ in range(k):
                P = bu(P, "Z")
            planes[(ry, rx)] = P
    for qy, qx in [(0, 0), (5, 11), (15, 15), (7, 2)]:
        S = sum(w[(a, b)] * roll(F, (qy + a, qx + b)) for a in (0, 1) for b in (0, 1))
        direct = S
        for _ in range(k):
            direct = bu(direct, "Z")
        via = sum(w[(a, b)] * roll(planes[((qy + a) % N % 2 ** k, (qx + b) % N % 2 ** k)],
                                   (((qy + a) % N) // 2 ** k, ((qx + b) % N) // 2 ** k))
                  for a in (0, 1) for b in (0, 1))
        assert np.array_equal(direct, via)
