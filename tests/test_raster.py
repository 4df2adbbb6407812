"""The GEMM tile raster (paper_2009_09523_b200/csrc/raster.cuh) is a bijection
onto the tile grid for every group height, and groups of gm rows are visited
column-major — checked on the host by compiling the header with g++."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

PROGRAM = r"""
#include <cstdio>
#include <vector>
#include "raster.cuh"
int main() {
  for (int tm_n = 1; tm_n <= 40; ++tm_n)
    for (int tn_n = 1; tn_n <= 40; ++tn_n)
      for (int gm = 0; gm <= 12; ++gm) {
        std::vector<int> seen(tm_n * tn_n, 0);
        int prev_m = -1, prev_n = -1;
        for (int t = 0; t < tm_n * tn_n; ++t) {
          int m, n;
          vntb::tc::tile_coords(t, tm_n, tn_n, gm, m, n);
          if (m < 0 || m >= tm_n || n < 0 || n >= tn_n || seen[m * tn_n + n]++) {
            std::printf("bad %d %d %d t=%d -> %d %d\n", tm_n, tn_n, gm, t, m, n);
            return 1;
          }
          // inside a group the row index advances fastest
          if (gm > 1 && t > 0 && (t % (gm * tn_n)) != 0 && n == prev_n && m != prev_m + 1) {
            std::printf("order %d %d %d t=%d\n", tm_n, tn_n, gm, t);
            return 1;
          }
          prev_m = m;
          prev_n = n;
        }
      }
  std::puts("ok");
  return 0;
}
"""


def test_tile_raster_is_a_bijection(tmp_path):
    src = tmp_path / "raster_test.cpp"
    exe = tmp_path / "raster_test"
    src.write_text(PROGRAM)
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT / 'paper_2009_09523_b200' / 'csrc'}",
                    "-o", str(exe), str(src)], check=True, timeout=120)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout + r.stderr
