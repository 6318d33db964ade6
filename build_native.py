"""Native build for every shared library in the repo (called by __graft_entry__.build()).

  synth/libdstack_synth_host.so   gcc  -- input generator, host build
  synth/libdstack_synth_dev.so    nvcc -- input generator, device build (sm_100a)
  oracle/liboracle.so             gcc  -- CPU oracle (test infrastructure)
  paper_2304_13541_b200/libdstack.so  nvcc -- the product: C-ABI + sm_100a kernels

Everything is built in-tree so the .so files travel to the GPU box with the repo snapshot.
Rebuilds only when a source is newer than the library (``force=True`` rebuilds all).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def build_synth(force=False):
    core = [os.path.join(ROOT, "synth", "synth_core.h"), os.path.join(ROOT, "include", "dstack_synth.h")]
    host_src = os.path.join(ROOT, "synth", "synth_host.c")
    host_out = os.path.join(ROOT, "synth", "libdstack_synth_host.so")
    if force or _stale(host_out, core + [host_src]):
        _run(["gcc", "-O2", "-std=c11", "-fopenmp", "-Wall", "-Wextra", "-shared", "-fPIC", host_src, "-o", host_out])
    dev_src = os.path.join(ROOT, "synth", "synth_dev.cu")
    dev_out = os.path.join(ROOT, "synth", "libdstack_synth_dev.so")
    if force or _stale(dev_out, core + [dev_src]):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", dev_src, "-o", dev_out])


def build_oracle(force=False):
    src = [os.path.join(ROOT, "oracle", "oracle.c"), os.path.join(ROOT, "oracle", "oracle.h")]
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, src):
        _run(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-Wall", "-Wextra", "-shared", "-fPIC", src[0], "-o", out])


def product_sources():
    csrc = os.path.join(ROOT, "paper_2304_13541_b200", "csrc")
    return sorted(glob.glob(os.path.join(csrc, "*.cu"))), sorted(glob.glob(os.path.join(csrc, "*.cuh")))


def build_product(force=False, verbose=False):
    cus, hdrs = product_sources()
    if not cus:
        return None
    out = os.path.join(ROOT, "paper_2304_13541_b200", "libdstack.so")
    deps = cus + hdrs + [os.path.join(ROOT, "include", "dstack.h"), os.path.join(ROOT, "synth", "synth_core.h")]
    if force or _stale(out, deps):
        log = _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC",
                    "-I", os.path.join(ROOT, "include"), *cus, "-o", out])
        if verbose:
            print(log)
        with open(os.path.join(ROOT, "paper_2304_13541_b200", "ptxas.log"), "w") as f:
            f.write(log)
    return out


def build_variant(out_name, defines):
    """Extra product build with -D flags (A/B experiments); never the default library."""
    cus, _ = product_sources()
    out = os.path.join(ROOT, "paper_2304_13541_b200", out_name)
    _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
          "-I", os.path.join(ROOT, "include"), *[f"-D{d}" for d in defines], *cus, "-o", out])
    return out


def build_all(force=False, verbose=False):
    build_synth(force)
    build_oracle(force)
    build_product(force, verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("ok")
