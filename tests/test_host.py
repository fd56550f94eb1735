"""CPU tests of the C-ABI library and the host logic (no GPU, no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_09165_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.load()


def _header_functions():
    src = open(os.path.join(ROOT, "include", "psd_filter.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(psd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib):
    from paper_2507_09165_b200 import _lib
    declared = _header_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == declared


def test_symbols_are_c_abi_and_kernels_are_sm100a(lib):
    out = os.popen(f"nm -D --defined-only {os.path.join(ROOT, 'paper_2507_09165_b200/lib/libpsdfilter.so')}").read()
    for name in _header_functions():
        assert re.search(rf"\bT {name}$", out, re.M), name        # unmangled extern "C"
    sass = os.popen("cuobjdump -sass " + os.path.join(ROOT, "paper_2507_09165_b200/lib/libpsdfilter.so") +
                    " 2>/dev/null | grep -cE 'UTCHMMA|UTMALDG|LDTM'").read().strip()
    if sass:
        assert int(sass) > 0, "tcgen05 / TMA instructions missing from the SASS"


def _create(lib, stages, eps=1e-3):
    from paper_2507_09165_b200 import filters
    deg, coef = filters.flatten(stages)
    h = ctypes.c_void_p()
    rc = lib.psd_filter_create(len(deg), (ctypes.c_int * len(deg))(*deg), (ctypes.c_double * len(coef))(*coef),
                               eps, ctypes.byref(h))
    return rc, h


def test_create_destroy_and_gemm_count(lib):
    """GEMM budget: 22 for T=7 d=5, 31 for T=10; NS-15 31, NS-10 21."""
    from paper_2507_09165_b200 import filters
    cases = [(filters.half_filter(), 22), (filters.single_filter(), 31),
             (filters.newton_schulz(15), 31), (filters.newton_schulz(10), 21), (filters.c2_filter(), 17),
             (filters.remez_half_prefix(6), 19), (filters.remez_half_prefix(3), 10)]
    for stages, g in cases:
        rc, h = _create(lib, stages)
        assert rc == 0
        assert lib.psd_filter_gemm_count(h, 1) == g
        assert lib.psd_filter_gemm_count(h, 0) == g - 1
        lib.psd_filter_destroy(h)
    rc, h = _create(lib, [(2.0,), (1.5, -0.5)])          # degree-1 stage = scalar, 0 GEMMs (R7)
    assert rc == 0 and lib.psd_filter_gemm_count(h, 1) == 3
    lib.psd_filter_destroy(h)
    lib.psd_filter_destroy(None)


def test_create_rejects_bad_arguments(lib):
    d = (ctypes.c_int * 1)(4)
    c = (ctypes.c_double * 3)(1.0, 2.0, 3.0)
    h = ctypes.c_void_p()
    assert lib.psd_filter_create(1, d, c, 1e-3, ctypes.byref(h)) == 1           # even degree
    assert b"odd" in lib.psd_last_error()
    d = (ctypes.c_int * 1)(3)
    assert lib.psd_filter_create(0, d, c, 1e-3, ctypes.byref(h)) == 1           # T < 1
    assert lib.psd_filter_create(1, d, c, 0.0, ctypes.byref(h)) == 1            # eps not in (0,1)
    c2 = (ctypes.c_double * 2)(1.0, float("nan"))
    assert lib.psd_filter_create(1, d, c2, 1e-3, ctypes.byref(h)) == 1          # non-finite
    assert lib.psd_filter_gemm_count(None, 1) == -1
    rc, h = _create(lib, [(1.5, -0.5)])
    assert lib.psd_filter_set_precision(h, 7) == 1
    assert lib.psd_filter_set_bound(h, 9) == 1
    assert lib.psd_filter_set_bound(h, 2) == 0                                   # PSD_BOUND_LANCZOS
    assert lib.psd_filter_set_lanczos(h, 0, 1.0) == 1                            # steps in [1, 64]
    assert lib.psd_filter_set_lanczos(h, 65, 1.0) == 1
    assert lib.psd_filter_set_lanczos(h, 20, 0.99) == 1                          # safety in [1, 2]
    assert lib.psd_filter_set_lanczos(h, 20, float("nan")) == 1
    assert lib.psd_filter_set_lanczos(h, 30, 1.02) == 0
    assert lib.psd_project(h, None, 4, 1, None, None) == 1                       # null pointers
    assert lib.psd_workspace_bytes(h, 4096, 32) > 6 * 32 * 4096 * 4096 * 2
    lib.psd_filter_destroy(h)


def test_product_tables_match_oracle_transcription():
    from oracle import tables
    from paper_2507_09165_b200 import filters
    assert np.array_equal(np.array(filters.HALF_REFINED), np.array(tables.F_HALF_REFINED))
    assert np.array_equal(np.array(filters.HALF), np.array(tables.F_HALF))
    assert np.array_equal(np.array(filters.SINGLE_REFINED), np.array(tables.F_SINGLE_REFINED))


def test_stabilization_fold_equals_literal_rescale():
    """Folding kappa into the next stage's coefficients (product side) is the same map as
    rescaling the iterate after each stage (oracle, literal P:L727), reading R1."""
    from oracle import chain, tables
    from paper_2507_09165_b200 import filters
    x = np.linspace(-1, 1, 20001)
    for folded, raw, kap in [(filters.half_filter(), tables.F_HALF_REFINED, tables.half_kappas()),
                             (filters.single_filter(), tables.F_SINGLE_REFINED, tables.single_kappas())]:
        a = chain.scalar_chain(x, folded)
        b = chain.scalar_chain(x, raw, kap)
        assert np.max(np.abs(a - b)) < 1e-13


def test_c2_coefficients_are_remez_output():
    """data/remez_filters.json was written by tools/make_coeffs.py from oracle.remez."""
    from oracle import remez
    from paper_2507_09165_b200 import filters
    st, _ = remez.sequential_remez(1e-3, [7] * 4)
    assert np.allclose(np.array(filters.c2_filter()), np.array(st), rtol=1e-12, atol=0)


def test_structured_torch_generator_matches_numpy():
    """synth.structured_torch (the n = 16384 input generator) gives the same fp32 values as
    synth.structured (same blocks, same butterflies)."""
    import numpy as np
    import synth
    torch = pytest.importorskip("torch")
    X, blocks = synth.structured(512, 9, block=64, family="sdp_shaped")
    Xt, blocks2 = synth.structured_torch(512, 9, block=64, family="sdp_shaped", device="cpu")
    assert np.array_equal(X, Xt.double().numpy())
    assert all(np.array_equal(a, b) for a, b in zip(blocks, blocks2))


def test_admm_and_peer_arguments_rejected_before_any_device_work(lib):
    """psd_admm_update and the peer-memory row-panel setup validate their arguments on the host
    (no GPU needed): bad sigma, aliasing, misalignment, unsupported shapes -> PSD_EINVAL /
    PSD_EUNSUPPORTED with a message."""
    from paper_2507_09165_b200 import filters
    rc, h = _create(lib, filters.half_filter())
    assert rc == 0
    fake = ctypes.c_void_p(0x10000)                      # 16-byte aligned, never dereferenced
    other = ctypes.c_void_p(0x20000)
    assert lib.psd_admm_update(h, fake, fake, None, -1.0, 64, 1, fake, other, None) == 1
    assert b"sigma" in lib.psd_last_error()
    assert lib.psd_admm_update(h, fake, fake, None, float("inf"), 64, 1, fake, other, None) == 1
    assert lib.psd_admm_update(h, fake, fake, None, 1.0, 64, 1, other, other, None) == 1      # S_out == X_out
    assert lib.psd_admm_update(h, fake, None, None, 1.0, 64, 1, fake, other, None) == 1       # null X_k
    assert lib.psd_admm_update(h, fake, ctypes.c_void_p(0x10004), None, 1.0, 64, 1, fake, other, None) == 1
    hb = ctypes.create_string_buffer(64)
    assert lib.psd_rowpanel_p2p_region(h, 1000, 3, 0, hb) == 1                 # n % nranks
    assert lib.psd_rowpanel_p2p_region(h, 1024, 16, 0, hb) == 1                # more than 8 ranks
    assert lib.psd_rowpanel_p2p_region(h, 1040, 2, 0, hb) == 1                 # rows per rank % 32
    assert lib.psd_rowpanel_p2p_region(h, 1024, 2, 2, hb) == 1                 # rank out of range
    assert lib.psd_rowpanel_p2p_attach(h, b"\0" * 128) == 1                    # no region yet
    assert lib.psd_project_rowpanel_p2p(h, fake, 1024, 0, 2, fake, 0, None) == 1
    assert lib.psd_filter_set_precision(h, 4) == 0                             # FP16X3
    assert lib.psd_rowpanel_p2p_region(h, 1024, 2, 0, hb) == 6                 # split: unsupported
    lib.psd_rowpanel_p2p_release(h)
    lib.psd_filter_destroy(h)


def test_coefficient_file_loader(tmp_path):
    """filters.load_coefficient_file (SPEC S:L213 layout): kappas folded offline equal the literal
    stabilisation of the oracle's scalar chain (reading R1/R7: a kappa after the last stage becomes a
    trailing degree-1 stage); inconsistent files are rejected."""
    import json
    import numpy as np
    from oracle import chain, tables
    from paper_2507_09165_b200 import filters
    kap = [1 / 1.01] * 6 + [0.99]
    path = tmp_path / "f.json"
    json.dump({"epsilon": 1e-3, "T": 7, "degrees": [5] * 7, "stages": [list(c) for c in tables.F_HALF_REFINED],
               "kappas": kap, "provenance": "test"}, open(path, "w"))
    stages, eps, prov = filters.load_coefficient_file(str(path))
    assert eps == 1e-3 and prov == "test" and len(stages) == 8 and stages[-1] == (0.99,)
    x = np.linspace(-1, 1, 10001)
    s_fold = chain.scalar_chain(x, stages)
    s_lit = chain.scalar_chain(x, tables.F_HALF_REFINED, kap)
    assert np.max(np.abs(s_fold - s_lit)) < 1e-13
    for bad in [{"T": 6}, {"degrees": [5] * 6 + [4]}, {"degrees": [3] * 7}]:
        d = {"epsilon": 1e-3, "T": 7, "degrees": [5] * 7, "stages": [list(c) for c in tables.F_HALF_REFINED]}
        d.update(bad)
        json.dump(d, open(path, "w"))
        with pytest.raises(ValueError):
            filters.load_coefficient_file(str(path))


@pytest.mark.parametrize("name", ["f_half_refined", "f_single_refined", "newton_schulz_10"])
def test_shipped_coefficient_files(name):
    """data/filters/*.json load to the filters the product path uses."""
    import os
    from paper_2507_09165_b200 import filters
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    stages, eps, _ = filters.load_coefficient_file(os.path.join(root, "data", "filters", name + ".json"))
    want = {"f_half_refined": filters.half_filter(), "f_single_refined": filters.single_filter(),
            "newton_schulz_10": filters.newton_schulz(10)}[name]
    assert stages == [tuple(c) for c in want]
