"""Generate data/SiC.tersoff -- a BUILDER FIXTURE, not a published file.

The reference ships only C.tersoff, so the two-species
table for BASELINE config 3 is composed from the Si(C) and C element sets with
chi_SiC = 0.9776 and these mixing rules (Tersoff 1989 style):
  entry (i,j,k): m=3, gamma=1, lambda3=0; c, d, h, eta, beta from element i;
  A_ij = sqrt(A_i A_j), B_ij = chi_ij sqrt(B_i B_j)  (chi=1 for i == j);
  lambda1, lambda2 = arithmetic means over the i-j pair;
  cutoff from the i-k pair: inner radius R-D and outer radius R+D each mixed
  geometrically, R = (in+out)/2, D = (out-in)/2 (i == k keeps the element's
  own R, D).
Both the B200 path and the oracle read this same file.
"""
import math
import os

EL = {  # A, B, lam1, lam2, beta, eta, c, d, h, R, D
    "Si": (1830.8, 471.18, 2.4799, 1.7322, 1.1e-6, 0.78734, 100390.0, 16.217, -0.59825, 2.85, 0.15),
    "C": (1393.6, 346.74, 3.4879, 2.2119, 1.5724e-7, 0.72751, 38049.0, 4.3484, -0.57058, 1.95, 0.15),
}
CHI = 0.9776


def entry(i, j, k):
    Ai, Bi, l1i, l2i, beta, eta, c, d, h, Ri, Di = EL[i]
    Aj, Bj, l1j, l2j = EL[j][:4]
    Rk, Dk = EL[k][9:11]
    chi = 1.0 if i == j else CHI
    A = math.sqrt(Ai * Aj)
    B = chi * math.sqrt(Bi * Bj)
    lam1 = 0.5 * (l1i + l1j)
    lam2 = 0.5 * (l2i + l2j)
    inner = math.sqrt((Ri - Di) * (Rk - Dk))
    outer = math.sqrt((Ri + Di) * (Rk + Dk))
    R = 0.5 * (inner + outer)
    D = 0.5 * (outer - inner)
    if i == k:  # same-element cutoff: the element's own R, D (no mixing noise)
        R, D = Ri, Di
    vals = [3, 1.0, 0.0, c, d, h, eta, beta, lam2, B, R, D, lam1, A]
    return " ".join([i, j, k] + [str(vals[0])] + [repr(float(v)) for v in vals[1:]])


def main():
    lines = ["# SiC two-species table: BUILDER FIXTURE composed by make_sic.py",
             "# (Si(C) + C 1988 element sets, chi_SiC = 0.9776, rules in make_sic.py).",
             "# Not a published parameter file; used identically by kernels and oracle.",
             "# elem_i elem_j elem_k  m gamma lambda3 c d h eta beta lambda2 B R D lambda1 A"]
    for i in ("Si", "C"):
        for j in ("Si", "C"):
            for k in ("Si", "C"):
                lines.append(entry(i, j, k))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "SiC.tersoff")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
