// sf_qtiles.cu -- Morton tiles of the pixel lattice for the tensor-core K~ build.
//
// K~ = F~ Q F~^H with Q = H H^T: k_ktilde_tc (sf_ktc.cu) works on
// tiles of <= 64 spatially adjacent pixels; each tile needs the union of its
// pixels' Q neighbourhoods.  Built once per engine on the host.
#include <algorithm>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// interleave the low 16 bits of v with zeros (Morton key)
static uint32_t spread16(uint32_t v) {
  v &= 0xFFFF;
  v = (v | (v << 8)) & 0x00FF00FF;
  v = (v | (v << 4)) & 0x0F0F0F0F;
  v = (v | (v << 2)) & 0x33333333;
  v = (v | (v << 1)) & 0x55555555;
  return v;
}

// Tiles of <= 64 pixels along the Morton order of the pixel lattice.
sf_status build_q_tiles(const double *xyz, int64_t n, const int64_t *qptr, const int32_t *qcol,
                        const double *qval, QTileHost &out) {
  if (n < 1 || n >= (1LL << 31)) return fail(SF_EINVAL, "Q tiles: size out of range");
  auto ranks = [&](int axis) {
    std::vector<double> u(n);
    for (int64_t p = 0; p < n; ++p) u[p] = xyz[3 * p + axis];
    std::vector<double> s(u);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    std::vector<uint32_t> r(n);
    for (int64_t p = 0; p < n; ++p)
      r[p] = (uint32_t)(std::lower_bound(s.begin(), s.end(), u[p]) - s.begin());
    return r;
  };
  const std::vector<uint32_t> rx = ranks(0), ry = ranks(1);
  std::vector<std::pair<uint64_t, int64_t>> key(n);
  for (int64_t p = 0; p < n; ++p)
    key[p] = {((uint64_t)(spread16(ry[p]) << 1 | spread16(rx[p])) << 32) | (uint64_t)p, p};
  std::sort(key.begin(), key.end());
  const int TP = 64;
  const int tiles = (int)((n + TP - 1) / TP);
  out.tiles = tiles;
  out.pix_off.assign(tiles + 1, 0);
  out.union_off.assign(tiles + 1, 0);
  out.pix_list.clear();
  out.union_list.clear();
  out.ent_off.assign(1, 0);
  out.ent_u.clear();
  out.ent_q.clear();
  out.max_union = 0;
  std::vector<int32_t> un;
  for (int t = 0; t < tiles; ++t) {
    const int64_t k0 = (int64_t)t * TP, k1 = std::min<int64_t>(n, k0 + TP);
    un.clear();
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t p = key[k].second;
      for (int64_t e = qptr[p]; e < qptr[p + 1]; ++e) un.push_back(qcol[e]);
    }
    std::sort(un.begin(), un.end());
    un.erase(std::unique(un.begin(), un.end()), un.end());
    if (un.size() > 32767) return fail(SF_EUNSUPPORTED, "Q tiles: neighbourhood too large");
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t p = key[k].second;
      out.pix_list.push_back((int32_t)p);
      for (int64_t e = qptr[p]; e < qptr[p + 1]; ++e) {
        out.ent_u.push_back((int16_t)(std::lower_bound(un.begin(), un.end(), qcol[e]) - un.begin()));
        out.ent_q.push_back(qval[e]);
      }
      out.ent_off.push_back((int32_t)out.ent_u.size());
    }
    out.union_list.insert(out.union_list.end(), un.begin(), un.end());
    out.pix_off[t + 1] = (int32_t)out.pix_list.size();
    out.union_off[t + 1] = (int32_t)out.union_list.size();
    out.max_union = std::max(out.max_union, (int)un.size());
  }
  out.mc = ((size_t)out.max_union * 16 * sizeof(double2) <= 100 * 1024) ? 16 : 8;
  if ((size_t)out.max_union * out.mc * sizeof(double2) > 200 * 1024)
    return fail(SF_EUNSUPPORTED, "Q tiles: neighbourhood too large for shared memory");
  return SF_OK;
}

}  // namespace sf
