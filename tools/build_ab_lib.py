"""Build an A/B variant of the library: the current csrc/ with some files
taken from another git revision, linked as
paper_2503_06433_b200/ab/libseesaw_b200_<tag>.so (in-tree, so it travels to
the GPU box; *.so is git-ignored).  Load it with SSB_LIB=<path> to time the
variant against the default library on the same box, e.g.

    python tools/build_ab_lib.py --rev 35a6953 --tag prev csrc/gemm_sm100.cu
    SSB_LIB=paper_2503_06433_b200/ab/libseesaw_b200_prev.so python tools/bench_decode.py --ab
"""
from __future__ import annotations

import argparse
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2503_06433_b200 import _build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rev", required=True)
ap.add_argument("--tag", required=True)
ap.add_argument("files", nargs="+", help="paths under paper_2503_06433_b200/ to take from --rev")
args = ap.parse_args()
tmp = Path(tempfile.mkdtemp(prefix="ssb_ab_"))
src = tmp / "csrc"
shutil.copytree(_build.CSRC, src)
for f in args.files:
    blob = subprocess.run(["git", "show", f"{args.rev}:paper_2503_06433_b200/{f}"], cwd=ROOT, check=True,
                          capture_output=True).stdout
    (tmp / f).write_bytes(blob)
flags = [c for c in _build.CFLAGS if not c.startswith("-I")] + [f"-I{_build.INCLUDE}", f"-I{src}"]


def cc(s: Path) -> Path:
    o = tmp / (s.stem + ".o")
    subprocess.run([_build.NVCC, *_build.ARCH, *flags, "-c", str(s), "-o", str(o)], check=True,
                   capture_output=True)
    return o


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(cc, sorted(src.glob("*.cu"))))
out = ROOT / "paper_2503_06433_b200" / "ab" / f"libseesaw_b200_{args.tag}.so"
out.parent.mkdir(exist_ok=True)
subprocess.run([_build.NVCC, *_build.ARCH, "-shared", "-o", str(out), *map(str, objs)], check=True)
print(out)
