"""tcgen05 / TMA evidence from the built engine's SASS (no GPU needed).

usage: python scripts/sass_evidence.py > profiles/r02_sass_tcgen05.md
Per GEMM kernel (EPI 0 fwd, 1 bwd-data, 2 dW; SPLIT 1 = 1-pass TF32 on fp32
operands, 3 = split-fp16 on kind::f16): counts of the tcgen05 MMA (UTCHMMA;
.2CTA = cta_group::2), TMA loads / stores (UTMALDG.2D/.3D, UTMASTG), TMEM
loads / stores (LDTM / STTM), tcgen05.commit (UTCBAR), packed fp16 converts
(F2FP) and the setmaxnreg role split, plus one sample line of each.
"""
import re
import subprocess
from collections import Counter, OrderedDict
from pathlib import Path

SO = Path(__file__).resolve().parents[1] / "paper_2009_09523_b200" / "libvnt_engine.so"
PAT = re.compile(r"\b(UTCHMMA(?:\.2CTA)?|UTMALDG\.[23]D(?:\.2CTA)?|UTMASTG\.[23]D|LDTM\.x\d+|STTM\.x\d+|"
                 r"UTCBAR(?:\.2CTA)?(?:\.MULTICAST)?|F2FP\.F16\.F32\.PACK|USETMAXREG\.[A-Z.]+)")
NAMES = {0: "fwd", 1: "bwd-data", 2: "dW"}


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True, check=True).stdout
    funcs = OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            k = re.search(r"k_gemm_tc(_pair)?ILi(\d)ELi(\d)E", name)
            cur = (("k_gemm_tc_pair" if k.group(1) else "k_gemm_tc"), int(k.group(2)), int(k.group(3))) if k else None
            if cur:
                funcs[cur] = (Counter(), {})
            continue
        if cur is None:
            continue
        for mn in PAT.findall(line):
            cnt, sample = funcs[cur]
            cnt[mn] += 1
            sample.setdefault(mn.split(".")[0], line.strip()[:110])
    print("# tcgen05 / TMA evidence in the built engine (round 2)\n")
    print("`cuobjdump -sass paper_2009_09523_b200/libvnt_engine.so` (built by `__graft_entry__.build()`, sm_100a), "
          "summarised by `scripts/sass_evidence.py`.  SPLIT 3 = the default split-fp16 operands on `kind::f16` "
          "(three MMAs per k16 step; `F2FP.F16.F32.PACK`: the epilogue's packed fp16 split; `UTMASTG`: the "
          "epilogue's TMA stores), SPLIT 1 = 1-pass TF32.\n")
    for (kern, epi, split), (cnt, sample) in sorted(funcs.items()):
        print(f"## `{kern}<{epi}, {split}>` ({NAMES[epi]}, {'split-fp16' if split == 3 else 'TF32'})\n")
        print(", ".join(f"`{k}` ×{v}" for k, v in sorted(cnt.items())) + "\n")
        print("```")
        for k in sorted(sample):
            print(sample[k])
        print("```\n")


if __name__ == "__main__":
    main()
