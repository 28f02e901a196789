"""Build libmarket_eq_b200.so in-tree for sm_100a (nvcc, no torch headers).

    python -m paper_2506_06258_b200._build [--verbose]

The k-section drop-in (ksection.cu) is compiled with --fmad=false so its
arithmetic rounds exactly like the reference's; the fast path may contract.
"""

import hashlib
import os
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libmarket_eq_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
          "--expt-relaxed-constexpr"]
SOURCES = {
    "abi.cu": [],
    "fast.cu": [],
    "reduce.cu": [],
    "generate.cu": ["--fmad=false"],
    "lifted.cu": [],
    "theory.cu": [],
    "ksection.cu": ["--fmad=false"],
}


def source_digest(extra_flags=()):
    """SHA-256 of everything the library is built from: every file of csrc/,
    the public header, the compiler and the flags.  Stored next to the
    library (`<lib>.sha256`) by build(); a prebuilt library is trusted only
    when its digest matches the sources it ships with (not their mtimes)."""
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        path = os.path.join(CSRC, name)
        if os.path.isfile(path):
            h.update(name.encode() + b"\0")
            with open(path, "rb") as fh:
                h.update(fh.read())
    with open(os.path.join(INCLUDE, "market_eq_b200.h"), "rb") as fh:
        h.update(fh.read())
    h.update(repr((NVCC, ARCH, COMMON, sorted(SOURCES.items()), list(extra_flags))).encode())
    return h.hexdigest()


def _digest_path(lib):
    return lib + ".sha256"


def up_to_date(lib=LIB, extra_flags=()):
    try:
        with open(_digest_path(lib)) as fh:
            return os.path.exists(lib) and fh.read().strip() == source_digest(extra_flags)
    except OSError:
        return False


def build(force=False, verbose=False, extra_flags=(), out=None):
    target = out or LIB
    if out is None and os.environ.get("MQ_LIB"):
        return os.environ["MQ_LIB"]  # a prebuilt variant was selected
    if not force and up_to_date(target, extra_flags):
        return target
    with tempfile.TemporaryDirectory() as tmp:
        objs = []
        for src, extra in SOURCES.items():
            obj = os.path.join(tmp, src + ".o")
            cmd = [NVCC, *ARCH, *COMMON, *extra, *extra_flags, "-c", os.path.join(CSRC, src),
                   "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            objs.append(obj)
        tmp_lib = os.path.join(tmp, "lib.so")
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", tmp_lib, *objs,
               "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        subprocess.run(cmd, check=True)
        os.replace(tmp_lib, target)
    with open(_digest_path(target), "w") as fh:
        fh.write(source_digest(extra_flags) + "\n")
    return target


if __name__ == "__main__":
    flags = ["-DMQ_PROFILE_WAITS"] if "--profile-waits" in sys.argv else []
    build(force=True, verbose="--verbose" in sys.argv, extra_flags=flags)
    print(LIB)
