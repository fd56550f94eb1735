"""Build libpsdfilter.so in-tree with nvcc for sm_100a.

    python -m paper_2507_09165_b200.build        # or __graft_entry__.build()

The library is a plain C-ABI shared object (include/psd_filter.h); CUDA runtime is
linked statically, the driver entry point for TMA descriptors is resolved at run time
(cudaGetDriverEntryPoint), so the .so only needs libcuda.so from the driver.
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libpsdfilter.so")
SOURCES = ["psd_api.cu", "sym_gemm.cu", "sym_gemm_2cta.cu", "bound_scale.cu", "small_batch.cu", "rowpanel.cu", "certificate.cu", "polar.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False, debug=False):
    """libpsdfilter.so; with debug=True libpsdfilter_dbg.so (-DPSD_DEBUG: the experiment switches
    and kernel phase stamps of DESIGN.md section 7, selected by PSD_LIB_VARIANT=debug)."""
    objdir = os.path.join(LIBDIR, "obj_dbg" if debug else "obj")
    lib = os.path.join(LIBDIR, "libpsdfilter_dbg.so") if debug else LIB
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "psd_filter.h"))
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append((src, [NVCC] + ARCH + FLAGS + (["-DPSD_DEBUG"] if debug else []) + ["-c", s, "-o", o]))
    # the translation units are independent: compile them concurrently
    procs = [(src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
             for src, cmd in jobs]
    failed = []
    for src, cmd, p in procs:
        out, err = p.communicate()
        if verbose or p.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + out + err)
        if p.returncode != 0:
            failed.append(src)
    if failed:
        raise RuntimeError("nvcc failed for " + ", ".join(failed))
    if force or _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return lib


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv, debug="--debug" in sys.argv))
