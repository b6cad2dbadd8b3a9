"""Host-side rotation helpers for scene generation and test fixtures
(src/rotation.cpp:7-77).  Not on the hot path: the device uses
csrc/detmath.cuh."""
from __future__ import annotations

import numpy as np


def skew(v) -> np.ndarray:
    x, y, z = v
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def rotation_matrix(r) -> np.ndarray:
    r = np.asarray(r, dtype=np.float64)
    t2 = float(r @ r)
    K = skew(r)
    if t2 < 1e-16:
        a, b = 1.0 - t2 / 6.0, 0.5 - t2 / 24.0
    else:
        t = np.sqrt(t2)
        a, b = np.sin(t) / t, (1.0 - np.cos(t)) / t2
    return np.eye(3) + a * K + b * (K @ K)


def rotation_log(R) -> np.ndarray:
    R = np.asarray(R, dtype=np.float64)
    tr = np.trace(R)
    if tr > 0.0:
        s = np.sqrt(tr + 1.0) * 2.0
        qw, qx, qy, qz = 0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s
    elif R[0, 0] >= R[1, 1] and R[0, 0] >= R[2, 2]:
        s = np.sqrt(max(0.0, 1.0 + R[0, 0] - R[1, 1] - R[2, 2])) * 2.0
        qw, qx, qy, qz = (R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s
    elif R[1, 1] >= R[2, 2]:
        s = np.sqrt(max(0.0, 1.0 + R[1, 1] - R[0, 0] - R[2, 2])) * 2.0
        qw, qx, qy, qz = (R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s
    else:
        s = np.sqrt(max(0.0, 1.0 + R[2, 2] - R[0, 0] - R[1, 1])) * 2.0
        qw, qx, qy, qz = (R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s
    qv = np.array([qx, qy, qz])
    if qw < 0.0:
        qw, qv = -qw, -qv
    nv = np.linalg.norm(qv)
    if nv < 1e-12:
        return 2.0 * qv
    return (2.0 * np.arctan2(nv, qw) / nv) * qv


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    while True:
        axis = rng.uniform(-1.0, 1.0, 3)
        if np.linalg.norm(axis) >= 1e-3:
            break
    return rotation_matrix(axis / np.linalg.norm(axis) * abs(rng.uniform(-1.0, 1.0)) * 3.0)
