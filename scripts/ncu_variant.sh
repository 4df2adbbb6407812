#!/bin/bash
# Per-launch duration of one kernel for engine builds with different defines
# (diagnostics, GPU box): scripts/ncu_variant.sh KERNEL_REGEX COUNT "DEFS" ["DEFS" ...]
set -e
K=$1; C=$2; shift 2
cp paper_2009_09523_b200/libvnt_engine.so /tmp/vnt_default.so
for D in "$@"; do
  python - "$D" <<'PY'
import subprocess, sys
sys.path.insert(0, ".")
from paper_2009_09523_b200 import build as b
subprocess.check_call([b.NVCC, *b.ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", *sys.argv[1].split(),
                       "-shared", "-o", "paper_2009_09523_b200/libvnt_engine.so", "paper_2009_09523_b200/csrc/engine.cu",
                       *b.nccl_flags(), "-lcuda"])
PY
  printf "%s: " "$D"
  ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$K" -c "$C" --csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra 2>/dev/null \
    | grep -v "^==" | tail -n +2 | awk -F'","' '{gsub(/"/,"",$NF); k=substr($5,1,40); s[k]+=$NF; n[k]++} END {for (k in s) printf "\n  %-40s %.1f us x %d", k, s[k]/n[k]/1000, n[k]; printf "\n"}'
done
cp /tmp/vnt_default.so paper_2009_09523_b200/libvnt_engine.so
