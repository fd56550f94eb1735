"""The rounding model behind the FP32-class parity bars (tools/rounding_model.py).

The north-star FP32 bar (1e-5) applies to the paper's filters (f~*_half, f~*_single).  Configs c1
(f*_half stages 1-3, sign error 0.86) and c2 (T = 4, d = 7, coefficients up to 128.8) amplify
rounding so strongly that even a TRUE float32 implementation of Algorithm 2 -- fp32 operands,
round-to-nearest fp32 accumulation -- misses 1e-5 against the float64 oracle; their bar is
therefore derived from this model (5e-5 ~ 2.5x the modelled fp32 worst case), not from the
north star.  No value here comes from the CUDA path."""
import numpy as np
import pytest

import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import rounding_model  # noqa: E402


def test_fp32_arithmetic_misses_1e5_on_c2_filter():
    e = rounding_model.model_errors("c2", 64, range(6), modes=("f32", "x3"))
    assert max(e["f32"]) > 1e-5            # infeasible for any FP32-class arithmetic
    assert max(e["f32"]) < 2.5e-5 and max(e["x3"]) < 2.5e-5   # the 5e-5 bar keeps 2x margin


def test_fp32_arithmetic_meets_1e5_on_paper_filters():
    for which, n in [("half", 64), ("single", 128)]:
        e = rounding_model.model_errors(which, n, range(3), modes=("f32", "x3"))
        assert max(e["f32"]) < 3e-6 and max(e["x3"]) < 2e-6, (which, e)


def test_model_exact_mode_is_the_oracle():
    """mode f64 of the emulation (same plan, float64) agrees with the oracle to 1e-12: the model
    differs from the oracle only by its rounding."""
    e = rounding_model.model_errors("half", 48, range(2), modes=("f64",))
    assert max(e["f64"]) < 1e-12
