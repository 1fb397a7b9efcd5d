"""In-tree build of the sm_100a planner library (and the test oracles).

    python -m paper_2503_06757_b200.build          # library only
    python -m paper_2503_06757_b200.build --all    # + oracle/ (and oracle/_ref when
                                                   #   /root/reference is present)

The library is a plain C-ABI shared object (include/prrtc_b200.h) built with
nvcc for sm_100a only; it lands in paper_2503_06757_b200/lib/ so it travels
with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libprrtc_b200.so"
SOURCES = ["prrtc_kernels.cu", "prrtc_capi.cu"]
HEADERS = ["prrtc_device.cuh", "prrtc_internal.h", "prrtc_launch.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 planner cannot be built")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False) -> Path:
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "prrtc_b200.h"]
    if not force and not _stale(LIB, deps):
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in SOURCES:
        obj = LIB_DIR / (Path(src).stem + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, f"-I{ROOT / 'include'}", f"-I{CSRC}", "-c",
               str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([nvcc, *ARCH, "-shared", "-o", str(tmp), *objs], check=True)
    os.replace(tmp, LIB)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return LIB


def build_oracle() -> None:
    """Checker libraries (test infrastructure): oracle/liboracle.so always,
    oracle/_ref/libprrtc_ref.so when the reference sources are present."""
    odir = ROOT / "oracle"
    subprocess.run(["make", "-s", "-C", str(odir), "liboracle.so"], check=True)
    if Path("/root/reference/proj/src").is_dir():
        subprocess.run(["make", "-s", "-j8", "-C", str(odir), "ref"], check=True)


def main(argv: list[str]) -> int:
    build_lib(force="--force" in argv, verbose="-v" in argv)
    if "--all" in argv:
        build_oracle()
    print(LIB)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
