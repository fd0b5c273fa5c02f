"""Builds the sm_100a shared library ``_build/libstmg_b200.so`` in-tree.

Each translation unit is compiled by ``nvcc -gencode arch=compute_100a,
code=sm_100a -lineinfo`` in parallel, then linked with ``-shared``. The
library exports exactly the C ABI of ``include/stmg_b200.h``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = BUILD / "libstmg_b200.so"

SOURCES = (["vmult.cu", "vanka.cu", "vanka_tc.cu", "aux_kernels.cu", "problems.cu", "stmg.cu", "setup.cpp", "st3d.cu", "setup3d.cpp", "stmg3d.cu", "comm_nccl.cpp", "patch3_gpu.cu"]
           + [f"vmult_r{r}s{s}.cu" for r in (1, 2, 3, 4) for s in (1, 2, 3, 4, 5)])
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the stmg_b200 CUDA library cannot be built")


def _host_cxx() -> list[str]:
    # nvcc must use the system g++ (the image's CXX points at a toolchain
    # without libgomp specs); pass it explicitly.
    gxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else (shutil.which("g++") or "g++")
    return ["-ccbin", gxx]


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + [Path(__file__)] + [ROOT / "include" / "stmg_b200.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    extra = os.environ.get("STMG_DEFS", "").split()  # experiment switches, e.g. -DSTMG_VMULT_SPLIT=1
    jobs = []
    for name in SOURCES:
        src = CSRC / name
        obj = BUILD / (name + ".o")
        if force or _stale(obj, src):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, *_host_cxx(), "-c", str(src), "-o", str(obj)]
            if name.endswith(".cpp"):
                cmd[1:1] = ["-x", "cu"]
            jobs.append((name, cmd))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            futs = {ex.submit(subprocess.run, cmd, capture_output=True, text=True): name for name, cmd in jobs}
            for fut in cf.as_completed(futs):
                res = fut.result()
                if verbose or res.returncode != 0:
                    sys.stderr.write(res.stdout + res.stderr)
                if res.returncode != 0:
                    raise RuntimeError(f"nvcc failed for {futs[fut]}")
    objs = [str(BUILD / (n + ".o")) for n in SOURCES]
    if force or jobs or not LIB.exists():
        cmd = [nvcc, *ARCH, *_host_cxx(), "-shared", "-o", str(LIB), *objs, "-lcudart", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link of libstmg_b200.so failed")
    # the drop-in command line (tools/stmg_cli.cpp: the reference's `stmg` flags on the GPU library)
    cli = BUILD / "stmg_gpu"
    src = ROOT / "tools" / "stmg_cli.cpp"
    if src.exists() and (force or not cli.exists() or cli.stat().st_mtime < max(src.stat().st_mtime,
                                                                              LIB.stat().st_mtime)):
        cuda_home = Path(_nvcc()).resolve().parents[1]
        gxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else "g++"
        cmd = [gxx, "-O2", "-std=c++17", "-I", str(ROOT / "include"), "-I", str(cuda_home / "include"), str(src),
               "-o", str(cli), "-L", str(BUILD), "-lstmg_b200", "-L", str(cuda_home / "lib64"), "-lcudart",
               f"-Wl,-rpath,$ORIGIN:{cuda_home / 'lib64'}"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("build of the stmg_gpu command line failed")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
