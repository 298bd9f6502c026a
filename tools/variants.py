"""Build experimental variants of libfc_b200.so with extra -D defines (A/B
experiments on the GPU box: run a diag tool with FC_LIB_PATH=<variant>).
Usage: python tools/variants.py name=DEF1,DEF2 [name2=...]
Outputs paper_2312_02493_b200/variants/libfc_<name>.so (git-ignored)."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_02493_b200 import build as b  # noqa: E402

outdir = b.PKG / "variants"
outdir.mkdir(exist_ok=True)
jobs = []
for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    jobs.append((outdir / f"libfc_{name}.so", tuple(d for d in defs.split(",") if d)))
with ThreadPoolExecutor(len(jobs) or 1) as ex:
    for p in ex.map(lambda j: b.build(out=j[0], defines=j[1]), jobs):
        print(p)
