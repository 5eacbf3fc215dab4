"""Synthetic DNN profiles (input recipe; DESIGN.md §Input recipe).

The paper profiles MobileNetV2 on an RTX 3090 (Fig. 3) and
counts per-sub-task workloads with torchsummaryX; neither data
set is published.  These profiles use standard-architecture MAC and output-
element counts at 224x224 (pools merged into the preceding sub-task) and the
paper's alpha/eta calibration definitions with Table I
values, plus an affine batch law d_n(b) = d_n(1)(1 + sigma(b-1)) that has the
Fig. 3 trends (total cost rising, per-sample cost falling with b).
"""
from __future__ import annotations

import numpy as np

# --- calibration constants --------------------------------------
F_MAX = 2.6e9          # Table I f_m,max
FE_MAX = 2.1e9         # Table I f_e,max
P_LOC = 11.0           # local inference power at f_max, W
SIGMA = 0.15           # batch-cost slope
ALPHA = 1.0            # Table I
ETA = 0.6              # Table I
B_MAX = 32
ACT_BITS = 8
INPUT_BITS = 224 * 224 * 3 * 8          # O_0 = 1,204,224 bits

MOBILENETV2_A = [10.84, 10.04, 29.2, 25.74, 15.47, 10.99, 10.99, 7.56, 10.31, 10.31, 10.31, 12.72,
                 22.69, 22.69, 15.61, 15.48, 15.48, 23.0, 21.35]
MOBILENETV2_O = [401.4, 200.7, 75.3, 75.3, 25.1, 25.1, 25.1, 12.5, 12.5, 12.5, 12.5, 18.8, 18.8, 18.8,
                 7.8, 7.8, 7.8, 15.7, 1.0]
VGG16_A = [86.7, 1849.7, 924.8, 1849.7, 924.8, 1849.7, 1849.7, 924.8, 1849.7, 1849.7, 462.4, 462.4,
           462.4, 102.8, 16.8, 4.1]
VGG16_O = [3211.3, 802.8, 1605.6, 401.4, 802.8, 802.8, 200.7, 401.4, 401.4, 100.4, 100.4, 100.4,
           25.1, 4.1, 4.1, 1.0]
RESNET18_A = [118.0, 1.8, 231.2, 231.2, 179.8, 231.2, 179.8, 231.2, 179.8, 231.2, 0.54]
RESNET18_O = [802.8, 200.7, 200.7, 200.7, 100.4, 100.4, 50.2, 50.2, 25.1, 25.1, 1.0]

# zeta: cycles per MAC such that MobileNetV2 (300.8 MMAC) runs in 3.2 ms at 2.6 GHz
# (beta = 2.13 <-> T = 10 ms, beta = 30.25 <-> T = 100 ms).
ZETA = 2.6e9 * 3.2e-3 / 300.8e6
# kappa from P = kappa f^3 / zeta at f_max.
KAPPA = P_LOC * ZETA / F_MAX ** 3


def _model(name, A_mmac, O_kelem, *, sigma=SIGMA, B_max=B_MAX, zeta=ZETA, kappa=KAPPA):
    from . import Model
    N = len(A_mmac)
    assert len(O_kelem) == N
    A = np.array([0.0] + [float(round(a * 1e6)) for a in A_mmac])
    O = np.array([float(INPUT_BITS)] + [float(round(o * 1e3)) * ACT_BITS for o in O_kelem])
    g = np.ones(N + 1)
    q = np.ones(N + 1)
    # alpha: edge batch-1 latency = local latency / alpha, both at max frequency
    d1 = zeta * FE_MAX / (ALPHA * F_MAX)
    # eta: local power / edge batch-1 power at max frequency:
    #   (c1/d1) fe_max^3 = (1/eta) (kappa/zeta) f_max^3
    c1 = d1 * (kappa / zeta) * F_MAX ** 3 / (ETA * FE_MAX ** 3)
    d = np.zeros((N + 1) * (B_max + 1))
    c = np.zeros((N + 1) * (B_max + 1))
    for n in range(1, N + 1):
        for b in range(1, B_max + 1):
            d[n * (B_max + 1) + b] = d1 * (1.0 + sigma * (b - 1))
            c[n * (B_max + 1) + b] = c1 * (1.0 + sigma * (b - 1))
    return Model(name, N, B_max, A, O, g, q, d, c)


def mobilenetv2(B_max=B_MAX):
    return _model("mobilenetv2", MOBILENETV2_A, MOBILENETV2_O, B_max=B_max)


def vgg16():
    return _model("vgg16", VGG16_A, VGG16_O)


def resnet18():
    return _model("resnet18", RESNET18_A, RESNET18_O)


def _toy(name, A, O, d12, c12):
    """Toys of SPEC.md:204 / SURVEY Appendix C: B_max = 2, g = q = 1."""
    from . import Model
    N = len(A) - 1
    B = 2
    d = np.zeros((N + 1) * (B + 1))
    c = np.zeros((N + 1) * (B + 1))
    for n in range(1, N + 1):
        d[n * (B + 1) + 1], d[n * (B + 1) + 2] = d12
        c[n * (B + 1) + 1], c[n * (B + 1) + 2] = c12
    return Model(name, N, B, np.array(A, float), np.array(O, float), np.ones(N + 1), np.ones(N + 1), d, c)


def toy1():
    return _toy("toy1", [0.0, 1e8, 2e8], [1e6, 4e5, 1e3], (0.8, 1.2), (2.5e-27, 4e-27))


def toy2():
    # "toy-2 = toy-1 with c scaled by 0.01"
    return _toy("toy2", [0.0, 1e8, 2e8], [1e6, 4e5, 1e3], (0.8, 1.2), (2.5e-29, 4e-29))


def toy4():
    # C1
    return _toy("toy4", [0.0, 1e8, 2e8, 2e8, 1e8], [1e6, 8e5, 4e5, 2e5, 1e3], (0.8, 1.2), (2.5e-29, 4e-29))
