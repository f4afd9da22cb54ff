"""The reduced (macromodel) system product, plainly.
TEST INFRASTRUCTURE ONLY.

PAPER.md eq. MV_product1: GMRES on eq. finalsystem needs

    (D - G^(E^,J^) T A^-1 B) Y,

computed "by first generating D, G, T, A and B, and then carrying out the
required matrix-vector multiplications", with G the AIM
operator (reading D1: G = -Z_eq).  Elements are the connected surfaces of the
mesh (oracle.precond.elements); element e of type d uses (D_d, T_d, A_d, B_d)
on its RWGs in ascending id.  Step by step for each element: b = B_d Y_e,
s = A_d^-1 b (numpy.linalg.solve, a library step), t_e = T_d s; then
y = Z_eq t (the oracle's AIM matvec); out_e = D_d Y_e - G t = D_d Y_e + y_e.
"""
from __future__ import annotations

import numpy as np


class ReducedSystem:
    def __init__(self, plan, elems, elem_type, blocks):
        """plan: oracle.aim.OraclePlan; elems: list of RWG-id arrays
        (oracle.precond.elements); elem_type[e]; blocks[d] = (D, T, A, B)."""
        self.plan = plan
        self.elems = elems
        self.elem_type = list(elem_type)
        self.blocks = blocks

    def apply_K(self, Y):
        Y = np.asarray(Y, dtype=np.complex128)
        t = np.zeros_like(Y)
        for idx, d in zip(self.elems, self.elem_type):
            D, T, A, B = self.blocks[d]
            t[idx] = T @ np.linalg.solve(A, B @ Y[idx])
        return t

    def apply_D(self, Y):
        Y = np.asarray(Y, dtype=np.complex128)
        out = np.zeros_like(Y)
        for idx, d in zip(self.elems, self.elem_type):
            out[idx] = self.blocks[d][0] @ Y[idx]
        return out

    def matvec(self, Y):
        """(D - G T A^-1 B) Y with G = -Z_eq (D1)."""
        return self.apply_D(Y) + self.plan.matvec(self.apply_K(Y))
