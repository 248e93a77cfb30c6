"""Build libpbnsim.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpbnsim.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "pbnsim.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple[str, ...] = (), out: str | None = None,
          extra: tuple[str, ...] = ()) -> str:
    """Compile libpbnsim.so (or, for A/B experiments, a variant `out` with extra -D defines).

    One nvcc per source file in parallel (host linkage only between the
    translation units), then one link step."""
    from concurrent.futures import ThreadPoolExecutor

    lib = os.path.join(HERE, out) if out else LIB
    if not force and not out and not _stale():
        return LIB
    tag = f"{os.path.basename(lib)}.{os.getpid()}"
    objdir = os.path.join(HERE, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", *[f"-D{d}" for d in defines], *extra,
              "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [_nvcc(), *common, "-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, r

    with ThreadPoolExecutor(max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, sources()))
    log_text = ""
    failed = None
    for src, obj, cmd, r in results:
        log_text += " ".join(cmd) + "\n" + r.stdout + r.stderr
        if r.returncode != 0 and failed is None:
            failed = (src, r)
    tmp = lib + f".tmp{os.getpid()}"
    if failed is None:
        cmd = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *[o for _, o, _, _ in results]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log_text += " ".join(cmd) + "\n" + r.stdout + r.stderr
        if r.returncode != 0:
            failed = ("link", r)
    log = os.path.join(HERE, "build.log" if not out else f"build_{out}.log")
    with open(log, "w") as f:
        f.write(log_text)
    shutil.rmtree(objdir, ignore_errors=True)
    if failed is not None:
        raise RuntimeError(f"nvcc failed on {failed[0]} (see {log}):\n{failed[1].stderr[-4000:]}")
    os.replace(tmp, lib)
    if verbose:
        print(log_text)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
