"""Build variant libraries for A/B runs: each NAME=FLAGS argument compiles the
whole library with extra nvcc flags into paper_1604_01713_b200/_lib/variants/
NAME.so; run with RG_LIB_PATH=<that .so>.

    python tools/ab_build.py w8r4="-DRG_V6_WARPS=8 -DRG_V6_RING=4" w4r6="-DRG_V6_WARPS=4 -DRG_V6_RING=6"
"""
import pathlib
import shlex
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

from paper_1604_01713_b200 import build as B  # noqa: E402

for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    out = B.LIB_DIR / "variants" / f"{name}.so"
    print(B.build(out=out, extra_flags=shlex.split(flags)))
