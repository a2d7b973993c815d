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


def _validation_error(msg: str) -> Exception:
    from .api import ValidationError
    return ValidationError(msg)


def directional_young(C: np.ndarray, axis: int) -> float:
    """props.hpp:61-65: E_a = 1 / S_aa along axis a in {1, 2, 3}."""
    if axis not in (1, 2, 3):
        raise _validation_error("axis must be 1, 2 or 3")
    return 1.0 / invert_tensor(C)[axis - 1, axis - 1]


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


def universal_anisotropy(C: np.ndarray) -> float:
    """props.hpp:94-97: A^U = 5 G_V / G_R + K_V / K_R - 6."""
    m = voigt_reuss_hill(C)
    return 5.0 * m["G_V"] / m["G_R"] + m["K_V"] / m["K_R"] - 6.0


def hs_bounds_two_phase(v: float, K1: float, G1: float, K2: float, G2: float):
    """props.hpp:101-118: Hashin-Shtrikman bounds with phase 1 (the stiffer) at fraction v."""
    if not (0.0 <= v <= 1.0):
        raise _validation_error("volume fraction must lie in [0, 1]")
    f1, f2 = v, 1.0 - v
    K = K1 if (f2 == 0.0 or K2 == K1) else K1 + f2 / (1.0 / (K2 - K1) + 3.0 * f1 / (3.0 * K1 + 4.0 * G1))
    if f2 == 0.0 or G2 == G1:
        G = G1
    else:
        zeta = G1 * (9.0 * K1 + 8.0 * G1) / (6.0 * (K1 + 2.0 * G1))
        G = G1 + f2 / (1.0 / (G2 - G1) + f1 / (G1 + zeta))
    return K, G


def hs_upper_bounds(v: float, E: float = 1.0, nu: float = 0.3):
    """props.hpp:121-125: solid/void composite at solid fraction v."""
    return hs_bounds_two_phase(v, E / (3.0 * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu)), 0.0, 0.0)


def offdiag_sum(C: np.ndarray) -> float:
    """props.hpp:127-132: sum of |C_ij| over the normal-shear block (i < 3 <= j)."""
    return float(np.abs(np.asarray(C, np.float64)[:3, 3:]).sum())


def isotropic_distance(C: np.ndarray) -> float:
    """props.hpp:137-158: Mandel-metric distance to the isotropic tensor with the
    Voigt moduli (the orthogonal projection onto the isotropic family)."""
    C = np.asarray(C, np.float64)
    Cd, Co, Cs = np.trace(C[:3, :3]), C[0, 1] + C[0, 2] + C[1, 2], np.trace(C[3:, 3:])
    K, G = (Cd + 2.0 * Co) / 9.0, (Cd - Co + 3.0 * Cs) / 15.0
    iso = np.zeros((6, 6))
    iso[:3, :3] = K - 2.0 * G / 3.0
    iso[np.arange(3), np.arange(3)] += 2.0 * G
    iso[np.arange(3, 6), np.arange(3, 6)] = G
    w = np.where(np.arange(6) >= 3, 2.0, 1.0)
    return float(np.sqrt((np.outer(w, w) * (C - iso) ** 2).sum()))


def make_report(C: np.ndarray, volume_ratio: float, E: float = 1.0, nu: float = 0.3) -> dict:
    """props.hpp:160-180."""
    C = np.asarray(C, np.float64)
    S = invert_tensor(C)
    m = voigt_reuss_hill(C)
    rep = {"E_x": 1.0 / S[0, 0], "E_y": 1.0 / S[1, 1], "E_z": 1.0 / S[2, 2], **m}
    rep["uai"] = universal_anisotropy(C)
    rep["offdiag"] = offdiag_sum(C)
    rep["volume_ratio"] = volume_ratio
    rep["K_HS_upper"], rep["G_HS_upper"] = hs_upper_bounds(volume_ratio, E, nu)
    rep["E_voigt"] = volume_ratio * E
    return rep


def csv_row(rep: dict | None) -> str:
    keys = CSV_HEADER.split(",")
    if rep is None:
        return ",".join(["nan"] * len(keys))
    return ",".join(repr(float(rep[k])) if not math.isnan(float(rep[k])) else "nan" for k in keys)
