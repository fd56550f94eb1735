"""ctypes binding of libpsdfilter.so (include/psd_filter.h).  Argument marshalling only:
every step of the projection runs in the library's CUDA kernels.

The library must have been built (``__graft_entry__.build()`` or
``python -m paper_2507_09165_b200.build``); there is no fallback of any kind.
"""
import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# PSD_LIB_VARIANT=debug selects libpsdfilter_dbg.so (build(debug=True)): the same sources with
# -DPSD_DEBUG, i.e. the experiment switches and kernel phase stamps; never used by tests or bench
LIB_PATH = os.path.join(_PKG, "lib", "libpsdfilter_dbg.so" if os.environ.get("PSD_LIB_VARIANT") == "debug"
                        else "libpsdfilter.so")

PSD_OK, PSD_EINVAL, PSD_ENOMEM, PSD_ECUDA, PSD_ENCCL, PSD_ENONFINITE, PSD_EUNSUPPORTED, PSD_ETIMEOUT = range(8)
STATUS_NAMES = {0: "PSD_OK", 1: "PSD_EINVAL", 2: "PSD_ENOMEM", 3: "PSD_ECUDA", 4: "PSD_ENCCL",
                5: "PSD_ENONFINITE", 6: "PSD_EUNSUPPORTED", 7: "PSD_ETIMEOUT"}
PRECISIONS = {"fp16": 0, "bf16": 1, "tf32": 2, "tf32x3": 3, "fp16x3": 4, "bf16x3": 5}
BOUNDS = {"frobenius": 0, "user": 1, "lanczos": 2}

# (name, restype, argtypes) for every symbol include/psd_filter.h declares.
_c = ctypes
SIGNATURES = [
    ("psd_version", _c.c_char_p, []),
    ("psd_last_error", _c.c_char_p, []),
    ("psd_filter_create", _c.c_int, [_c.c_int, _c.c_void_p, _c.c_void_p, _c.c_double, _c.POINTER(_c.c_void_p)]),
    ("psd_filter_destroy", None, [_c.c_void_p]),
    ("psd_filter_set_precision", _c.c_int, [_c.c_void_p, _c.c_int]),
    ("psd_filter_set_bound", _c.c_int, [_c.c_void_p, _c.c_int]),
    ("psd_filter_set_lanczos", _c.c_int, [_c.c_void_p, _c.c_int, _c.c_double]),
    ("psd_filter_set_accum_chunk", _c.c_int, [_c.c_void_p, _c.c_int64]),
    ("psd_filter_gemm_count", _c.c_int, [_c.c_void_p, _c.c_int]),
    ("psd_project", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p]),
    ("psd_sign", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p]),
    ("psd_polar", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p,
                             _c.c_void_p, _c.c_void_p]),
    ("psd_polar_rect", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_int64, _c.c_void_p,
                                  _c.c_void_p, _c.c_void_p, _c.c_void_p]),
    ("psd_project_ex", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p,
                                  _c.c_void_p, _c.c_int, _c.c_void_p]),
    ("psd_admm_update", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_double, _c.c_int64,
                                   _c.c_int64, _c.c_void_p, _c.c_void_p, _c.c_void_p]),
    ("psd_filter_certificate", _c.c_int, [_c.c_void_p, _c.POINTER(_c.c_double), _c.POINTER(_c.c_double),
                                          _c.POINTER(_c.c_double), _c.POINTER(_c.c_double)]),
    ("psd_status", _c.c_int, [_c.c_void_p, _c.c_void_p]),
    ("psd_workspace_bytes", _c.c_int64, [_c.c_void_p, _c.c_int64, _c.c_int64]),
    ("psd_profile", _c.c_int, [_c.c_void_p, _c.c_int]),
    ("psd_profile_read", _c.c_int, [_c.c_void_p, _c.POINTER(_c.c_double), _c.POINTER(_c.c_int64),
                                    _c.POINTER(_c.c_int64)]),
    ("psd_project_host", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_int,
                                    _c.c_void_p]),
    ("psd_nccl_unique_id", _c.c_int, [_c.c_char_p]),
    ("psd_nccl_comm_create", _c.c_int, [_c.c_char_p, _c.c_int, _c.c_int, _c.POINTER(_c.c_void_p)]),
    ("psd_nccl_comm_destroy", _c.c_int, [_c.c_void_p]),
    ("psd_project_rowpanel", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int, _c.c_int, _c.c_void_p,
                                        _c.c_int, _c.c_void_p, _c.c_void_p]),
    ("psd_project_rowpanel_virtual", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int, _c.c_void_p,
                                                _c.c_int, _c.c_void_p]),
    ("psd_rowpanel_p2p_region", _c.c_int, [_c.c_void_p, _c.c_int64, _c.c_int, _c.c_int, _c.c_char_p]),
    ("psd_rowpanel_p2p_attach", _c.c_int, [_c.c_void_p, _c.c_char_p]),
    ("psd_project_rowpanel_p2p", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int, _c.c_int, _c.c_void_p,
                                            _c.c_int, _c.c_void_p]),
    ("psd_project_rowpanel_p2p_virtual", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int, _c.c_void_p,
                                                    _c.c_int, _c.c_void_p]),
    ("psd_rowpanel_p2p_timeout", _c.c_int, [_c.c_void_p, _c.c_double]),
    ("psd_rowpanel_p2p_release", None, [_c.c_void_p]),
    ("psd_rowpanel_tiles", _c.c_int, [_c.c_int64, _c.c_int, _c.c_int, _c.c_void_p, _c.c_int]),
    ("psd_sym_product", _c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_double, _c.c_double,
                                   _c.c_int64, _c.c_int64, _c.c_void_p, _c.c_void_p]),
]

_lib = None


class PsdError(RuntimeError):
    def __init__(self, code, where):
        msg = load().psd_last_error().decode()
        super().__init__(f"{where}: {STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def load():
    """Load the library (raises if it was not built: no CPU or PyTorch fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (CUDA path is mandatory)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def check(code, where):
    if code != PSD_OK:
        raise PsdError(code, where)
