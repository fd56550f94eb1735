"""Composite-filter coefficient sets and the stabilisation fold (product side).

Coefficients are offline inputs of the hot path (BASELINE.json north_star).  The
paper's Tables 1-2 are transcribed here independently of ``oracle/`` (the two
sides share no tables); ``tests/test_host.py`` checks the transcriptions agree.

Stage t is f_t(x) = sum_j c_{t,j} x^{2j+1}, f_1 applied first.
"""
import json
import os

# Table 2 right column, f~*_half: the half-precision filter, T = 7, d = 5.
HALF_REFINED = (
    (8.2885332412, -22.5927099246, 15.8201383114),
    (4.1666196466, -2.9679004036, 0.5307623217),
    (4.0611848147, -2.9698947955, 0.5492133813),
    (3.6678301399, -2.7561018955, 0.5421513305),
    (2.7632556383, -2.0607754898, 0.4695405857),
    (2.0527445797, -1.4345145882, 0.4070669182),
    (1.8804816691, -1.2583997294, 0.3779501813),
)
# Table 2 left column, f*_half: Remez, eps = 1e-3.
HALF = (
    (8.4703288038, -25.1080747067, 18.6292755991),
    (4.1828341833, -3.1087011099, 0.5806066814),
    (3.9618572790, -2.9540637464, 0.5629761180),
    (3.2865862170, -2.4647201345, 0.5073576939),
    (2.2737499945, -1.6446603679, 0.4161909275),
    (1.8887161973, -1.2651572253, 0.3765189256),
    (1.8750008858, -1.2500009843, 0.3750000984),
)
# Table 1 right column, f~*_single: the single-precision filter, T = 10.
SINGLE_REFINED = (
    (8.3119043343, -23.0739115930, 16.4664144722),
    (4.1439360087, -2.9176674704, 0.5246212487),
    (4.0257813209, -2.9025002398, 0.5334261214),
    (3.5118574347, -2.5740236523, 0.5050097282),
    (2.4398158400, -1.7586675341, 0.4191290613),
    (1.9779835097, -1.3337358510, 0.3772169049),
    (1.9559726949, -1.3091355170, 0.3746734515),
    (1.9282822454, -1.2823649693, 0.3704626545),
    (1.9220135179, -1.2812524618, 0.3707011753),
    (1.8942192942, -1.2613293407, 0.3676616051),
)
# Newton-Schulz stage 1.5 x - 0.5 x^3.
NEWTON_SCHULZ = (1.5, -0.5)


def fold_stabilization(stages, kappa, n_scaled):
    """Fold the stabilisation rescale of P:L727 into the coefficients.

    Reading R1: X <- kappa X after stage t for t = 1..n_scaled (never after
    the last stage).  kappa after stage t equals feeding kappa Z into stage t+1:
    f_{t+1}(kappa Z) = sum_j c_{t+1,j} kappa^{2j+1} Z^{2j+1}.
    """
    out = [list(c) for c in stages]
    T = len(out)
    for t in range(min(n_scaled, T - 1)):
        nxt = out[t + 1]
        for j in range(len(nxt)):
            nxt[j] = nxt[j] * kappa ** (2 * j + 1)
    return [tuple(c) for c in out]


def fold_kappas(stages, kappas):
    """Per-stage stabilisation factors kappa_t (X <- kappa_t X after stage t) folded into
    the coefficients: kappa_t for t < T into stage t + 1 (as ``fold_stabilization``); a kappa after
    the last stage, if not 1, stays a trailing degree-1 stage (reading R7: a scalar, 0 products)."""
    out = [list(c) for c in stages]
    T = len(out)
    if len(kappas) != T:
        raise ValueError("one kappa per stage")
    for t in range(T - 1):
        k = float(kappas[t])
        if k != 1.0:
            out[t + 1] = [v * k ** (2 * j + 1) for j, v in enumerate(out[t + 1])]
    stages = [tuple(c) for c in out]
    if float(kappas[-1]) != 1.0:
        stages.append((float(kappas[-1]),))
    return stages


def load_coefficient_file(path):
    """A coefficient file (the JSON layout of SPEC S:L213: {"epsilon", "T", "degrees", "stages":
    [[c_1, c_3, c_5, ...], ...], "provenance"}, optional "kappas": one stabilisation factor per
    stage, folded offline by ``fold_kappas``).  Third-party sets (e.g. Polar Express)
    are ingested this way.  Returns (stages, eps, provenance); raises ValueError on an
    inconsistent file."""
    with open(path) as f:
        d = json.load(f)
    stages = [tuple(float(v) for v in c) for c in d["stages"]]
    T = int(d.get("T", len(stages)))
    degrees = [int(x) for x in d.get("degrees", [2 * len(c) - 1 for c in stages])]
    if T != len(stages) or len(degrees) != T:
        raise ValueError(f"{path}: T, degrees and stages disagree")
    for t, (deg, c) in enumerate(zip(degrees, stages)):
        if deg % 2 == 0 or deg < 1 or len(c) != (deg + 1) // 2:
            raise ValueError(f"{path}: stage {t}: degree {deg} with {len(c)} coefficients")
    eps = float(d.get("epsilon", d.get("eps", 1e-3)))
    if "kappas" in d:
        stages = fold_kappas(stages, d["kappas"])
    return stages, eps, d.get("provenance", "")


def half_filter():
    """f~*_half with 1/1.01 after stages 1..6 (the 16-bit path)."""
    return fold_stabilization(HALF_REFINED, 1.0 / 1.01, 6)


def single_filter():
    """f~*_single with 1/1.001 after stages 1..8 (the FP32 path)."""
    return fold_stabilization(SINGLE_REFINED, 1.0 / 1.001, 8)


def remez_half_prefix(T):
    """First T stages of f*_half: the eps=1e-3 sequential-Remez chain of length T
    (Algorithm 1 is greedy, so its T-stage output is the prefix; configs c1 (T=3), c3 (T=6))."""
    return [tuple(c) for c in HALF[:T]]


def remez_filter_file(key):
    """Coefficient sets written offline by tools/make_coeffs.py (data/remez_filters.json)."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "remez_filters.json")
    with open(path) as f:
        d = json.load(f)[key]
    return [tuple(c) for c in d["stages"]], d["eps"]


def c2_filter():
    """Config c2: T = 4 stages of degree 7, eps = 1e-3 (Remez, Appendix-B tool)."""
    return remez_filter_file("c2_T4_d7_eps1e-3")[0]


def newton_schulz(iterations):
    return [NEWTON_SCHULZ] * iterations


def flatten(stages):
    """(degrees, coeffs) in the ABI layout of psd_filter_create."""
    degrees = [2 * len(c) - 1 for c in stages]
    coeffs = [float(v) for c in stages for v in c]
    return degrees, coeffs
