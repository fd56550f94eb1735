"""Offline coefficient tool: writes the coefficient sets the paper does not print.

Calls ONLY ``oracle/`` (Algorithm 1 sequential Remez, + App. A).
The output JSON files under ``data/`` are inputs of both the CUDA path and the
oracle (coefficients are offline inputs per BASELINE.json north_star).

    python tools/make_coeffs.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import certify, remez  # noqa: E402


def main():
    out = {}
    # Config c2: T = 4 stages of degree 7, eps = 1e-3 (BASELINE.json configs[1]).
    st, iv = remez.sequential_remez(1e-3, [7] * 4)
    out["c2_T4_d7_eps1e-3"] = {
        "cite": "Algorithm 1 (P:L523-545) with App. A Remez (P:L1037-1081); eps=1e-3, d_t=7, T=4",
        "eps": 1e-3, "degrees": [7] * 4, "stages": [list(c) for c in st],
        "intervals": [list(v) for v in iv],
        "sign_err_on_eps1": certify.sign_err(st, 1e-3)[0],
        "relu_err": certify.relu_err(st)[0],
    }
    path = os.path.join(ROOT, "data", "remez_filters.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
