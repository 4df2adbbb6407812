"""A/B timing of engine build variants on one GPU box (diagnostics).

Builds libvnt_engine.so once per variant (extra nvcc defines), then runs
bench.py round-robin (A, B, ..., A, B, ...) so clock / power drift hits every
variant alike, and prints the median ms/step per variant.  Leaves the default
build in place at the end.

usage: python scripts/ab_bench.py ROUNDS "name=DEFS" ["name=DEFS" ...] [-- bench args]
  e.g. python scripts/ab_bench.py 3 "base=" "nbuf2=-DVNT_DW_NBUF=2"
"""
import json
import shutil
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2009_09523_b200 import build as b  # noqa: E402

PKG = ROOT / "paper_2009_09523_b200"
SO = PKG / "libvnt_engine.so"


def build(defs, out):
    subprocess.check_call([b.NVCC, *b.ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", *defs,
                           "-shared", "-o", str(out), str(PKG / "csrc" / "engine.cu"), *b.nccl_flags(), "-lcuda"])


def main():
    args = sys.argv[1:]
    extra = []
    if "--" in args:
        i = args.index("--")
        args, extra = args[:i], args[i + 1:]
    rounds = int(args[0])
    variants = []
    for spec in args[1:]:
        name, _, defs = spec.partition("=")
        out = Path(f"/tmp/vnt_ab_{name}.so")
        build(defs.split(), out)
        variants.append((name, out))
    shutil.copy(SO, "/tmp/vnt_ab_default.so")
    res = {n: [] for n, _ in variants}
    for r in range(rounds):
        for name, so in variants:
            shutil.copy(so, SO)
            out = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "3", "--no-cpu-baseline",
                                  "--no-extra", *extra], cwd=ROOT, capture_output=True, text=True, timeout=900).stdout
            d = json.loads(out.strip().splitlines()[-1])
            res[name].append(d["ms_per_step"])
            print(f"round {r} {name:>10}: {d['ms_per_step']:.3f} ms/step ({d['value']:.4g} samples/s, "
                  f"sm {d['clocks'].get('sm_mhz')} MHz)", flush=True)
    shutil.copy("/tmp/vnt_ab_default.so", SO)
    for name, v in res.items():
        print(f"{name:>10}: median {statistics.median(v):.3f} ms/step over {len(v)}")


if __name__ == "__main__":
    main()
