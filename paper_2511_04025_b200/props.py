"""Scalar properties of an effective tensor (props.hpp:1-182, host post-processing).

Restates `make_report` for the sweep outputs: directional Young's moduli,
Voigt/Reuss/Hill moduli, universal anisotropy index, normal-shear coupling,
Hashin-Shtrikman upper bounds for a solid/void composite, Voigt bound.
"""
from __future__ import annotations

import math

import numpy as np

CSV_HEADER = ("E_x,E_y,E_z,K_V,K_R,G_V,G_R,K_eff,G_eff,E_eff,uai,offdiag,volume_ratio,"
              "K_HS_upper,G_HS_upper,E_voigt")


class SingularTensorError(ValueError):
    pass


def invert_tensor(C: np.ndarray) -> np.ndarray:
    """props.hpp:51-55 (FullPivLU invertibility check)."""
    C = np.asarray(C, np.float64)
    if np.linalg.matrix_rank(C) < 6:
        raise SingularTensorError("elastic tensor is singular")
    return np.linalg.inv(C)


def voigt_reuss_hill(C: np.ndarray) -> dict:
    """props.hpp:71-92."""
    S = invert_tensor(C)
    Cd, Co, Cs = C[0, 0] + C[1, 1] + C[2, 2], C[0, 1] + C[0, 2] + C[1, 2], C[3, 3] + C[4, 4] + C[5, 5]
    Sd, So, Ss = S[0, 0] + S[1, 1] + S[2, 2], S[0, 1] + S[0, 2] + S[1, 2], S[3, 3] + S[4, 4] + S[5, 5]
    K_V, G_V = (Cd + 2.0 * Co) / 9.0, (Cd - Co + 3.0 * Cs) / 15.0
    K_R, G_R = 1.0 / (Sd + 2.0 * So), 15.0 / (4.0 * Sd - 4.0 * So + 3.0 * Ss)
    K, G = 0.5 * (K_V + K_R), 0.5 * (G_V + G_R)
    return dict(K_V=K_V, K_R=K_R, G_V=G_V, G_R=G_R, K_eff=K, G_eff=G, E_eff=9 * K * G / (3 * K + G))


def hs_upper_bounds(v: float, E: float = 1.0, nu: float = 0.3):
    """props.hpp:103-127 with phase 2 = void."""
    K1, G1 = E / (3.0 * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))
    f1, f2 = v, 1.0 - v
    if f2 == 0.0:
        return K1, G1
    K = K1 + f2 / (1.0 / (0.0 - K1) + 3.0 * f1 / (3.0 * K1 + 4.0 * G1))
    zeta = G1 * (9.0 * K1 + 8.0 * G1) / (6.0 * (K1 + 2.0 * G1))
    G = G1 + f2 / (1.0 / (0.0 - G1) + f1 / (G1 + zeta))
    return K, G


def make_report(C: np.ndarray, volume_ratio: float, E: float = 1.0, nu: float = 0.3) -> dict:
    """props.hpp:160-180."""
    C = np.asarray(C, np.float64)
    S = invert_tensor(C)
    m = voigt_reuss_hill(C)
    rep = {"E_x": 1.0 / S[0, 0], "E_y": 1.0 / S[1, 1], "E_z": 1.0 / S[2, 2], **m}
    rep["uai"] = 5.0 * m["G_V"] / m["G_R"] + m["K_V"] / m["K_R"] - 6.0
    rep["offdiag"] = float(np.abs(C[:3, 3:]).sum())
    rep["volume_ratio"] = volume_ratio
    rep["K_HS_upper"], rep["G_HS_upper"] = hs_upper_bounds(volume_ratio, E, nu)
    rep["E_voigt"] = volume_ratio * E
    return rep


def csv_row(rep: dict | None) -> str:
    keys = CSV_HEADER.split(",")
    if rep is None:
        return ",".join(["nan"] * len(keys))
    return ",".join(repr(float(rep[k])) if not math.isnan(float(rep[k])) else "nan" for k in keys)
