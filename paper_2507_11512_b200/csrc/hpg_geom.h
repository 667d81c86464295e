// Structural arithmetic of one rank-level, shared by host and device.
//
// Everything the reference computes at setup with Python loops -- greedy
// coloring, the (color, natural) permutation, the compacted 27-point ELL rows,
// halo slots and send lists -- has a closed form on the structured grid:
//
//  * color(x,y,z)   = parity bits of the axes with extent >= 2
//                     (ref: coloring.py:49-55 greedy first-fit on a 27-pt lattice)
//  * iperm(x,y,z)   = color_offset[c] + (x>>1) + hx*((y>>1) + hy*(z>>1))
//                     (ref: coloring.py:78-80, rows sorted by (color, natural))
//  * ELL row        = in-domain neighbours in z-slowest/x-fastest offset order,
//                     compacted, padded to 27 (ref: problem.py:88-142)
//  * halo slot      = n + base(neighbour) + natural position inside the
//                     face/edge/corner region, neighbours by ascending rank
//                     (ref: comm.py:180-236)
//
// The same functions build the device ELL (hpg_build kernels) and the host
// export used by the CPU parity tests, so the two can never drift apart.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HPG_HD __host__ __device__ __forceinline__
#else
#define HPG_HD inline
#endif

namespace hpg {

constexpr int kWidth = 27;
constexpr int kDiagSlot = 13;  // (0,0,0) in offset order
constexpr int kMaxColors = 27; // first-fit on a 27-point lattice never needs more

struct Geom {
  int lx, ly, lz;        // local extent
  int ox, oy, oz;        // global origin of this rank's box
  int gx, gy, gz;        // global extent
  int ncolors;
  int bit[3];            // parity bit of each axis in the color id, -1 if extent < 2
  int64_t n;             // owned rows
  int64_t off[kMaxColors + 1];  // color block offsets (ncolors+1 used)
  // General (e.g. JPL) colorings: explicit tables instead of the greedy closed
  // form (device pointers; null for greedy).  perm: new row -> natural row,
  // iperm: natural row -> new row (ref: coloring.py:78-80).
  const int32_t* perm_tab;
  const int32_t* iperm_tab;
  int64_t halo_base[27]; // per face/edge/corner (index of offset), -1 if no neighbour
  int64_t halo_size;
  int nbr_rank[27];      // rank id of the neighbour across each face/edge/corner, -1 if none
};

HPG_HD int offset_index(int dx, int dy, int dz) { return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1); }

HPG_HD int color_of(const Geom& g, int x, int y, int z) {
  int c = 0;
  if (g.bit[0] >= 0) c |= (x & 1) << g.bit[0];
  if (g.bit[1] >= 0) c |= (y & 1) << g.bit[1];
  if (g.bit[2] >= 0) c |= (z & 1) << g.bit[2];
  return c;
}

// natural local coords -> color-permuted row
HPG_HD int64_t iperm(const Geom& g, int x, int y, int z) {
  if (g.iperm_tab) return g.iperm_tab[x + (int64_t)g.lx * (y + (int64_t)g.ly * z)];
  const int c = color_of(g, x, y, z);
  const int64_t hx = (g.lx - (x & 1) + 1) >> 1;
  const int64_t hy = (g.ly - (y & 1) + 1) >> 1;
  return g.off[c] + (x >> 1) + hx * ((int64_t)(y >> 1) + hy * (int64_t)(z >> 1));
}

// color-permuted row -> natural local coords
HPG_HD void decode(const Geom& g, int64_t i, int& x, int& y, int& z) {
  if (g.perm_tab) {
    const int64_t nat = g.perm_tab[i];
    x = (int)(nat % g.lx);
    y = (int)((nat / g.lx) % g.ly);
    z = (int)(nat / ((int64_t)g.lx * g.ly));
    return;
  }
  int c = 0;
  while (c + 1 < g.ncolors && i >= g.off[c + 1]) ++c;
  const int px = g.bit[0] >= 0 ? (c >> g.bit[0]) & 1 : 0;
  const int py = g.bit[1] >= 0 ? (c >> g.bit[1]) & 1 : 0;
  const int pz = g.bit[2] >= 0 ? (c >> g.bit[2]) & 1 : 0;
  const int64_t hx = (g.lx - px + 1) >> 1;
  const int64_t hy = (g.ly - py + 1) >> 1;
  int64_t pos = i - g.off[c];
  const int64_t X = pos % hx;
  pos /= hx;
  const int64_t Y = pos % hy;
  const int64_t Z = pos / hy;
  x = (int)(2 * X + px);
  y = (int)(2 * Y + py);
  z = (int)(2 * Z + pz);
}

// One compacted ELL row.  val codes: 26 on the diagonal, -1 off it.
// Returns nnz; *diag receives the diagonal's slot.  Off-rank neighbours get
// their halo slot.  Padding is left to the caller.
HPG_HD int build_row(const Geom& g, int64_t i, int32_t* cols, double* vals, int* diag) {
  int x, y, z;
  decode(g, i, x, y, z);
  int s = 0;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int ax = x + dx, ay = y + dy, az = z + dz;
        const int wx = ax + g.ox, wy = ay + g.oy, wz = az + g.oz;
        if (wx < 0 || wx >= g.gx || wy < 0 || wy >= g.gy || wz < 0 || wz >= g.gz) continue;
        const int sx = ax < 0 ? -1 : (ax >= g.lx ? 1 : 0);
        const int sy = ay < 0 ? -1 : (ay >= g.ly ? 1 : 0);
        const int sz = az < 0 ? -1 : (az >= g.lz ? 1 : 0);
        int64_t col;
        if (sx == 0 && sy == 0 && sz == 0) {
          col = iperm(g, ax, ay, az);
        } else {
          const int64_t rw = sx == 0 ? g.lx : 1;
          const int64_t rh = sy == 0 ? g.ly : 1;
          const int64_t p = (sx == 0 ? ax : 0) + rw * ((sy == 0 ? ay : 0) + rh * (int64_t)(sz == 0 ? az : 0));
          col = g.halo_base[offset_index(sx, sy, sz)] + p;
        }
        const bool self = dx == 0 && dy == 0 && dz == 0;
        if (self) *diag = s;
        cols[s] = (int32_t)col;
        vals[s] = self ? 26.0 : -1.0;
        ++s;
      }
  return s;
}

// Number of points of the send (inside) or halo (outside) region across
// face/edge/corner (sx, sy, sz).
HPG_HD int64_t region_size(const Geom& g, int sx, int sy, int sz) {
  return (int64_t)(sx == 0 ? g.lx : 1) * (sy == 0 ? g.ly : 1) * (sz == 0 ? g.lz : 1);
}

// p-th point (natural order) of the inside region next to face (sx,sy,sz),
// as a permuted local row: the send list the peer requests (ref: comm.py:209-217).
HPG_HD int64_t send_row(const Geom& g, int sx, int sy, int sz, int64_t p) {
  const int64_t rw = sx == 0 ? g.lx : 1;
  const int64_t rh = sy == 0 ? g.ly : 1;
  const int px = (int)(p % rw);
  const int py = (int)((p / rw) % rh);
  const int pz = (int)(p / (rw * rh));
  const int x = sx == 0 ? px : (sx > 0 ? g.lx - 1 : 0);
  const int y = sy == 0 ? py : (sy > 0 ? g.ly - 1 : 0);
  const int z = sz == 0 ? pz : (sz > 0 ? g.lz - 1 : 0);
  return iperm(g, x, y, z);
}

// Does row i read any halo slot?  (row lies on a face that has a neighbour)
HPG_HD bool row_has_halo(const Geom& g, int64_t i) {
  int x, y, z;
  decode(g, i, x, y, z);
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int ax = x + dx, ay = y + dy, az = z + dz;
        const int sx = ax < 0 ? -1 : (ax >= g.lx ? 1 : 0);
        const int sy = ay < 0 ? -1 : (ay >= g.ly ? 1 : 0);
        const int sz = az < 0 ? -1 : (az >= g.lz ? 1 : 0);
        if ((sx | sy | sz) != 0 && g.halo_base[offset_index(sx, sy, sz)] >= 0) return true;
      }
  return false;
}

}  // namespace hpg
