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
HEADERS = ["prrtc_device.cuh", "prrtc_internal.h", "prrtc_launch.h", "prrtc_warp.cuh"]
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


REF_INCLUDE = Path("/root/reference/proj/include")
REF_SRC = Path("/root/reference/proj/src")
DROPIN_LIB = LIB_DIR / "libprrtc_b200_dropin.so"
DEMO_BIN = ROOT / "tests" / "cpp" / "bin" / "dropin_demo"
REF_SOURCES = ["collision", "geometry", "kernels", "kernels_scalar", "kernels_avx2", "kinematics", "nn",
               "planner", "sampling"]


def build_dropin(force: bool = False) -> Path | None:
    """C++ drop-in prrtc::b200::plan (reference types) + its demo/test binary.
    Both compile against the reference's headers, so they are built only
    where /root/reference exists; the outputs travel with the repo snapshot."""
    if not REF_INCLUDE.is_dir():
        return None
    cxx = shutil.which("g++") or "g++"
    dsrc = PKG / "dropin" / "prrtc_dropin.cpp"
    deps = [dsrc, PKG / "dropin" / "prrtc_dropin.hpp", ROOT / "include" / "prrtc_b200.h", LIB]
    flags = ["-std=c++20", "-O2", "-fPIC", f"-I{REF_INCLUDE}", f"-I{ROOT / 'include'}", f"-I{PKG / 'dropin'}"]
    if force or _stale(DROPIN_LIB, deps):
        subprocess.run([cxx, *flags, "-shared", "-o", str(DROPIN_LIB), str(dsrc), f"-L{LIB_DIR}",
                        "-lprrtc_b200", "-Wl,-rpath,$ORIGIN"], check=True)
    demo = ROOT / "tests" / "cpp" / "dropin_demo.cpp"
    if REF_SRC.is_dir() and (force or _stale(DEMO_BIN, [demo, DROPIN_LIB])):
        DEMO_BIN.parent.mkdir(parents=True, exist_ok=True)
        # reference sources compiled in place (never copied), -mavx2 as the
        # reference's AVX2 kernels require
        srcs = [str(REF_SRC / f"{s}.cpp") for s in REF_SOURCES]
        subprocess.run([cxx, *flags, "-mavx2", "-ffp-contract=off", f"-I{REF_SRC}", "-o", str(DEMO_BIN),
                        str(demo), *srcs, f"-L{LIB_DIR}", "-lprrtc_b200_dropin", "-lprrtc_b200",
                        f"-Wl,-rpath,{LIB_DIR}", "-Wl,-rpath,$ORIGIN/../../../paper_2503_06757_b200/lib",
                        "-lpthread"], check=True)
    return DROPIN_LIB


def build_oracle() -> None:
    """Checker libraries (test infrastructure): oracle/liboracle.so always,
    oracle/_ref/libprrtc_ref.so when the reference sources are present."""
    odir = ROOT / "oracle"
    subprocess.run(["make", "-s", "-C", str(odir), "liboracle.so"], check=True)
    if Path("/root/reference/proj/src").is_dir():
        subprocess.run(["make", "-s", "-j8", "-C", str(odir), "ref"], check=True)


def main(argv: list[str]) -> int:
    build_lib(force="--force" in argv, verbose="-v" in argv)
    build_dropin(force="--force" in argv)
    if "--all" in argv:
        build_oracle()
    print(LIB)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
