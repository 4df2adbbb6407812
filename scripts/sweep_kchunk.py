"""K-chunk promotion sweep (GPU box): cfg3 samples/s (bench.py, short run) and
the headline-width gradient deviation (scripts/diag_headline.py) for each
(VNT_TC_KFIRST, VNT_TC_KCHUNK).  usage: python scripts/sweep_kchunk.py kf:kc ..."""
import json
import os
import re
import subprocess
import sys

for spec in sys.argv[1:]:
    kf, kc = spec.split(":")
    env = dict(os.environ, VNT_TC_KFIRST=kf, VNT_TC_KCHUNK=kc)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "20", "--warmup", "3", "--no-cpu-baseline",
                          "--no-extra"], env=env, capture_output=True, text=True, timeout=600).stdout
    d = json.loads(out.strip().splitlines()[-1])
    diag = subprocess.run([sys.executable, "scripts/diag_headline.py", "auto"], env=env, capture_output=True,
                          text=True, timeout=600).stdout
    devs = [float(m) for m in re.findall(r"max dev ([0-9.e+-]+)", diag)] or [float("nan")]
    loss = re.search(r"loss ([0-9.]+) ([0-9.]+)", diag)
    print(f"kfirst {kf:>5} kchunk {kc:>4}: {d['value']:.4g} samples/s, {d['ms_per_step']:.3f} ms/step, "
          f"frac {d['roofline']['frac']:.3f} | grad dev (masks resolved) {max(devs):.2e} of max, "
          f"loss {loss.group(1)} vs {loss.group(2)}", flush=True)
