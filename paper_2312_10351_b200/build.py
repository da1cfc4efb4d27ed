"""Build libopara.so in-tree with nvcc for sm_100a.

    python -m paper_2312_10351_b200.build        # incremental
    python -m paper_2312_10351_b200.build --clean

Every .cpp/.cu under csrc/ is compiled to build/*.o (in parallel) and linked
into paper_2312_10351_b200/libopara.so, which travels to the GPU box with the
repo snapshot.  Host C++ is compiled with -ffp-contract=off (bit-exact
dominant_share, see csrc/sched.cpp).
"""

from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
_FLAGS = os.environ.get("OPARA_NVCC_FLAGS", "")  # A/B experiments only: own object dir + relink
BUILD = ROOT / "build" / ("opara" if not _FLAGS else "opara-" + hashlib.sha1(_FLAGS.encode()).hexdigest()[:8])
LIB = PKG / "libopara.so"
STAMP = PKG / "libopara.hash"   # source hash of the linked libopara.so (travels with it)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", f"-I{ROOT / 'include'}", f"-I{CSRC}",
          "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "--expt-relaxed-constexpr",
          *_FLAGS.split()]


def _sources() -> list[Path]:
    return sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.cpp")])


def _headers() -> list[Path]:
    return sorted([*CSRC.glob("*.h"), *CSRC.glob("*.cuh"), *(ROOT / "include").glob("*.h")])


def source_hash() -> str:
    """sha1 (12 hex) of every source and header the library is built from plus
    the extra nvcc flags; embedded in opara_version() and checked on load."""
    h = hashlib.sha1(_FLAGS.encode())
    for f in _sources() + _headers():
        h.update(f.name.encode() + b"\0" + f.read_bytes() + b"\0")
    return h.hexdigest()[:12]


def _compile(src: Path, verbose: bool, src_hash: str) -> Path:
    obj = BUILD / (src.name + ".o")
    stamp = BUILD / (src.name + ".hash")
    # content-addressed: an object is reused only if it was built from exactly
    # these sources (mtimes lie after checkouts and snapshot copies)
    key = src_hash if src.name == "sched.cpp" else hashlib.sha1(
        b"".join(f.read_bytes() for f in [src] + _headers()) + _FLAGS.encode()).hexdigest()
    if obj.exists() and stamp.exists() and stamp.read_text() == key:
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.name == "sched.cpp":
        cmd.append(f'-DOPARA_SOURCE_HASH="{src_hash}"')
    if src.suffix == ".cu":
        cmd += ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "c++"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
    if verbose and res.stderr:
        (BUILD / (src.name + ".ptxas.txt")).write_text(res.stderr)
    stamp.write_text(key)
    return obj


def build(verbose: bool = False, clean: bool = False) -> Path:
    if clean and BUILD.exists():
        shutil.rmtree(BUILD)
    BUILD.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    src_hash = source_hash()
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as pool:
        objs = list(pool.map(lambda s: _compile(s, verbose, src_hash), srcs))
    if LIB.exists() and STAMP.exists() and STAMP.read_text() == src_hash:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    STAMP.write_text(src_hash)
    return LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true", help="keep ptxas -v reports in build/")
    args = ap.parse_args(argv)
    lib = build(verbose=args.verbose, clean=args.clean)
    print(lib)
    return 0


if __name__ == "__main__":
    sys.exit(main())
