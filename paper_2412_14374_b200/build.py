"""In-tree build of libpp200.so (sm_100a) with nvcc.

Run ``python -m paper_2412_14374_b200.build`` or ``__graft_entry__.build()``.
Objects go to ``build/``; the shared library lands next to this file so it
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import shutil
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent
CSRC = HERE / "csrc"
BUILD = ROOT / "build" / "pp200"
LIB = HERE / "libpp200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-I", str(ROOT / "include"), "-I", str(CSRC)]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (2.28.x)
        base = pathlib.Path(list(nn.__path__)[0])
        inc, lib = base / "include", base / "lib"
        if (inc / "nccl.h").exists() and (lib / "libnccl.so.2").exists():
            return inc, lib
    except Exception:
        pass
    return None, None


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return cand


def sources():
    return sorted(CSRC.glob("*.cu"))


def _compile(src: pathlib.Path, extra: list[str]) -> pathlib.Path:
    obj = BUILD / (src.stem + ".o")
    deps = [src] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "pp200.h"]
    if obj.exists() and all(obj.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return obj
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> pathlib.Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    inc, lib = _nccl_dirs()
    extra = ["-I", str(inc)] if inc else []
    if inc:
        extra.append("-DPP200_HAVE_NCCL=1")
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra), srcs))
    link = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
    if lib:
        link += ["-L", str(lib), "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print(f"built {LIB} from {len(srcs)} sources")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
