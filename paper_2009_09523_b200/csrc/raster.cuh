// Tile raster of the persistent tcgen05 GEMMs (also compiled by the host
// unit test tests/test_raster.py, hence plain C++ when not under nvcc).
//
// Tile t of a tiles_m x tiles_n grid maps to (tm, tn): groups of gm tile rows,
// column-major inside a group, so the tiles resident at once (CTA b takes
// tiles b, b + grid, ...) share A and B operand panels in L2.  gm <= 1 is the
// plain row-major order.  A bijection onto the grid for every gm.
#pragma once

#if defined(__CUDACC__)
#define VNT_RASTER_FN __host__ __device__ __forceinline__
#else
#define VNT_RASTER_FN inline
#endif

namespace vntb {
namespace tc {

VNT_RASTER_FN void tile_coords(int tile, int tiles_m, int tiles_n, int gm, int& tm, int& tn) {
  if (gm <= 1) {
    tm = tile / tiles_n;
    tn = tile % tiles_n;
    return;
  }
  const int per_group = gm * tiles_n;
  const int g = tile / per_group;
  const int first = g * gm;
  const int rows = tiles_m - first < gm ? tiles_m - first : gm;
  const int t = tile - g * per_group;
  tm = first + t % rows;
  tn = t / rows;
}

}  // namespace tc
}  // namespace vntb
