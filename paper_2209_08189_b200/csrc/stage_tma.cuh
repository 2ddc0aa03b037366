// Shared-memory-staged semi-Lagrangian sweeps (tricubic / trilinear).
//
// Why: the direct gather (interp.cuh, gather_lean) reads its 64 taps per point
// with scalar LDGs whose warp requests straddle two L1 lines; the sweep runs at
// ~70 % of the L1 data pipe (ncu: l1tex__data_pipe_lsu_wavefronts ~4 per point)
// and is L1-bound, not HBM-bound.  Here one CTA owns a tile of arrival voxels
// (one x1 plane, TJ x2 rows, TK x3 voxels), reduces the floor-index bounding box
// of the tile's departure points, and copies that source box -- stencil
// included -- into shared memory with bulk asynchronous copies
// (cp.async.bulk, one per box row, completion on an mbarrier).  The copy
// engine writes shared memory without touching registers or the LSU pipe; the
// taps are then 4 conflict-free LDS.32 per stencil row (one 32-bit address add
// per row, immediate tap offsets).
//
// Smooth characteristics keep the box small (C2 256^3: ~6 x 9 x 140 floats =
// 30 KB for 512 points).  A tile whose box exceeds the shared-memory budget
// (rough or huge displacements), or that holds a non-finite displacement,
// takes the direct gather -- same taps, same arithmetic order, same results.
//
// Arithmetic is gather_lean's (lagrange4 weights, z taps FMA-chained, then y,
// then x), so results equal the direct gather's up to FMA contraction.
#pragma once
#include <climits>
#include "interp.cuh"

namespace vr {
namespace stg {

constexpr int NT = 128;                 // threads per CTA

// Tile / residency configuration: PPT points per thread (tile = PPT * NT
// points), box budget per CTA, CTAs per SM the launch bounds aim for.  (PPT = 2
// with 24 KB boxes and 9 CTAs / SM measured 6 % slower: the halo share of the
// box grows faster than residency helps.)
template <int PPT_, int BUDGET_KB = 36, int CTAS = 6, bool PAD32 = true> struct Cfg {
  static constexpr int PPT = PPT_;
  static constexpr int kSmemBudget = BUDGET_KB * 1024;
  static constexpr int kCtas = CTAS;
  // box row pitch: a multiple of 32 floats (PAD32) or the copied length (a
  // multiple of 4) nudged off multiples of 32 -- a smaller box, more CTAs / SM
  static constexpr bool kPad32 = PAD32;
};
// residency variants (vr_set_gather_mode 1 / 2 / 3)
using CfgA = Cfg<4, 36, 6, true>;
using CfgB = Cfg<4, 30, 7, false>;
using CfgC = Cfg<4, 27, 8, false>;
using CfgD = Cfg<4, 36, 6, false>;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}

__device__ __forceinline__ int floor4(int a) { return a & ~3; }   // floor to a multiple of 4 (two's complement)

// tile geometry: TK x3 voxels (a multiple of 32, <= NT) by TJ = PPT * NT / TK x2 rows
struct Tile {
  int tk, tj;
};
inline Tile tile_for(const Dims& d, int ppt) {
  const int tk = d.n3 >= NT ? NT : d.n3;
  return Tile{tk, ppt * (NT / tk)};
}
inline bool staged_ok(const Dims& d) { return d.n3 % 32 == 0 && d.n2 >= 4; }

struct Box {
  int x0, y0, s;       // first plane / row (unwrapped) and first x3 voxel (multiple of 4, unwrapped)
  int nx, ny, len;     // planes, rows, floats copied per row (multiple of 4)
  int pitch;           // shared-memory row stride (multiple of 32 floats)
  int ok;
};

// Per-point stencil base / fraction of one tile point (split_coord + the slab clamp).
template <int ORDER, bool SLAB>
struct PointSplit {
  int b1, b2, b3;
  float t1, t2, t3;
  bool bad;
  __device__ __forceinline__ PointSplit(const PlaneSrc<1, SLAB>& src, const Dims& d, int i, int j, int k, float d1,
                                        float d2, float d3) {
    // huge displacements need gather_disp_lean's per-point pre-wrap
    bad = !(isfinite(d1) && isfinite(d2) && isfinite(d3) && (SLAB || fabsf(d1) < d.n1 - 4) &&
            fabsf(d2) < d.n2 - 4 && fabsf(d3) < d.n3 - 4);
    split_coord(i, d1, b1, t1);
    split_coord(j, d2, b2, t2);
    split_coord(k, d3, b3, t3);
    if (SLAB) b1 = ORDER == ORDER_CUBIC ? clampi(b1, 1 - src.w, src.L1 + src.w - 3) : clampi(b1, -src.w, src.L1 + src.w - 2);
  }
};

// One CTA = one tile (TJ x2 rows x TK x3 voxels of one x1 plane), PPT points
// per thread:
//   1. load the tile's displacements, reduce the stencil bounds (warp
//      reductions + one CTA exchange) -> box of source rows;
//   2. thread 0 arms the mbarrier with the box byte count, warp 0 issues one
//      bulk copy per box row (two where the x3 segment wraps);
//   3. wait on the mbarrier, gather the tile's points from shared memory.
// Phases of one CTA are serial; the ~6 CTAs resident per SM overlap each
// other's copy latency.  (Measured alternatives on B200 -- persistent CTAs with
// displacement prefetch, double-buffered boxes behind CTA barriers, and a
// warp-specialised producer/consumer pipeline -- were all slower: the extra
// buffer halves the resident CTAs, and occupancy is what hides the gather's
// shared-memory latency.)  A box over budget, or a tile with a non-finite or
// huge displacement, gathers directly.  ORDER: ORDER_CUBIC or ORDER_LINEAR;
// epi(idx, v) writes voxel idx.
template <int ORDER, bool SLAB, class Epi, class CF>
__global__ void __launch_bounds__(NT, CF::kCtas) sweep_kernel(PlaneSrc<1, SLAB> src, Dims d,
                                                              const float* __restrict__ disp, Tile T, int x0,
                                                              Epi epi) {
  constexpr int PPT = CF::PPT;
  constexpr int kSmemBudget = CF::kSmemBudget;
  constexpr int LO = ORDER == ORDER_CUBIC ? 1 : 0;   // stencil reach below / above the base index
  constexpr int HI = ORDER == ORDER_CUBIC ? 2 : 1;
  extern __shared__ __align__(128) float box[];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ int red[NT / 32][7];
  __shared__ Box bx;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) mbar_init(smem_u32(&bar), 1);
  const int64_t N = d.n();
  const int ntk = (d.n3 + T.tk - 1) / T.tk;
  const int tile_j = blockIdx.x / ntk, tile_k = blockIdx.x - tile_j * ntk;
  const int i = (int)blockIdx.y + x0;
  const int kk = tid % T.tk, jr = tid / T.tk, rstep = NT / T.tk;
  const int k = tile_k * T.tk + kk;
  float dv[3][PPT];
  bool valid[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int j = tile_j * T.tj + jr + rstep * p;
    valid[p] = k < d.n3 && j < d.n2;
    const int id = valid[p] ? (i * d.n2 + j) * d.n3 + k : 0;
    dv[0][p] = valid[p] ? __ldg(disp + id) : 0.f;
    dv[1][p] = valid[p] ? __ldg(disp + N + id) : 0.f;
    dv[2][p] = valid[p] ? __ldg(disp + 2 * N + id) : 0.f;
  }
  int mn1 = INT_MAX, mx1 = INT_MIN, mn2 = INT_MAX, mx2 = INT_MIN, mn3 = INT_MAX, mx3 = INT_MIN;
  bool bad = false;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if (!valid[p]) continue;
    const PointSplit<ORDER, SLAB> ps(src, d, i, tile_j * T.tj + jr + rstep * p, k, dv[0][p], dv[1][p], dv[2][p]);
    bad |= ps.bad;
    mn1 = min(mn1, ps.b1); mx1 = max(mx1, ps.b1);
    mn2 = min(mn2, ps.b2); mx2 = max(mx2, ps.b2);
    mn3 = min(mn3, ps.b3); mx3 = max(mx3, ps.b3);
  }
  mn1 = __reduce_min_sync(~0u, mn1); mx1 = __reduce_max_sync(~0u, mx1);
  mn2 = __reduce_min_sync(~0u, mn2); mx2 = __reduce_max_sync(~0u, mx2);
  mn3 = __reduce_min_sync(~0u, mn3); mx3 = __reduce_max_sync(~0u, mx3);
  const int anybad = __any_sync(~0u, bad);
  if (lane == 0) {
    red[wid][0] = mn1; red[wid][1] = mx1; red[wid][2] = mn2; red[wid][3] = mx2;
    red[wid][4] = mn3; red[wid][5] = mx3; red[wid][6] = anybad;
  }
  __syncthreads();   // also publishes the mbarrier init
  if (tid == 0) {
    int a0 = INT_MAX, a1 = INT_MIN, c0 = INT_MAX, c1 = INT_MIN, e0 = INT_MAX, e1 = INT_MIN, bb = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
      a0 = min(a0, red[w][0]); a1 = max(a1, red[w][1]);
      c0 = min(c0, red[w][2]); c1 = max(c1, red[w][3]);
      e0 = min(e0, red[w][4]); e1 = max(e1, red[w][5]);
      bb |= red[w][6];
    }
    Box b;
    b.x0 = a0 - LO;
    b.nx = a1 - a0 + LO + HI + 1;
    b.y0 = c0 - LO;
    b.ny = c1 - c0 + LO + HI + 1;
    b.s = floor4(e0 - LO);
    b.len = ((e1 + HI + 1 - b.s) + 3) & ~3;
    // row pitch a multiple of 32 floats: lanes of a warp split across two box
    // rows / planes still hit disjoint banks
    if (CF::kPad32) b.pitch = (b.len + 31) & ~31;
    else b.pitch = (b.len & 31) == 0 ? b.len + 4 : b.len;
    b.ok = !bb && a0 <= a1 && b.len <= d.n3 && b.ny <= d.n2 && (SLAB || b.nx <= d.n1) &&
           (int64_t)b.nx * b.ny * b.pitch * 4 <= kSmemBudget;
    if (b.ok) mbar_expect_tx(smem_u32(&bar), (unsigned)(b.nx * b.ny * b.len * 4));
    bx = b;
  }
  __syncthreads();
  const Box b = bx;
  if (!b.ok) {   // direct per-point gather (same taps, same arithmetic order)
#pragma unroll 1
    for (int p = 0; p < PPT; ++p) {
      const int j = tile_j * T.tj + jr + rstep * p;
      if (k >= d.n3 || j >= d.n2) continue;
      const int id = (i * d.n2 + j) * d.n3 + k;
      float o;
      gather_disp_lean<ORDER, 1, SLAB>(src, d, i, j, k, __ldg(disp + id), __ldg(disp + N + id),
                                       __ldg(disp + 2 * N + id), &o);
      epi(id, o);
    }
    return;
  }
  if (wid == 0) {
    const int psz = d.n2 * d.n3;
    const int nrows = b.nx * b.ny;
    int s = b.s % d.n3;
    if (s < 0) s += d.n3;
    const int first = min(b.len, d.n3 - s);   // floats before the x3 wrap
    const unsigned bar_a = smem_u32(&bar);
    for (int r = lane; r < nrows; r += 32) {
      const int xr = r / b.ny, yr = r - xr * b.ny;
      int x = b.x0 + xr;
      if (!SLAB) x = wrap1(x, d.n1);
      int y = (b.y0 + yr) % d.n2;
      if (y < 0) y += d.n2;
      const float* row = src.plane(0, x, psz) + y * d.n3;
      const unsigned dst = smem_u32(box + r * b.pitch);
      bulk_g2s(dst, row + s, (unsigned)first * 4u, bar_a);
      if (first < b.len) bulk_g2s(dst + first * 4u, row, (unsigned)(b.len - first) * 4u, bar_a);
    }
  }
  mbar_wait(smem_u32(&bar), 0);
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if (!valid[p]) continue;
    const int j = tile_j * T.tj + jr + rstep * p;
    const PointSplit<ORDER, SLAB> ps(src, d, i, j, k, dv[0][p], dv[1][p], dv[2][p]);
    float o;
    if (ORDER == ORDER_CUBIC) {
      float wx[4], wy[4], wz[4];
      lagrange4(ps.t1, wx);
      lagrange4(ps.t2, wy);
      lagrange4(ps.t3, wz);
      const int xs = b.ny * b.pitch;
      const float* base = box + ((ps.b1 - 1 - b.x0) * b.ny + (ps.b2 - 1 - b.y0)) * b.pitch + (ps.b3 - 1 - b.s);
      float acc = 0.0f;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        float sa = 0.0f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float* r = base + a * xs + c * b.pitch;
          const float sb = wz[0] * r[0] + wz[1] * r[1] + wz[2] * r[2] + wz[3] * r[3];
          sa += wy[c] * sb;
        }
        acc += wx[a] * sa;
      }
      o = acc;
    } else {
      const float* r0 = box + ((ps.b1 - b.x0) * b.ny + (ps.b2 - b.y0)) * b.pitch + (ps.b3 - b.s);
      const float* r1 = r0 + b.pitch;
      const float* r2 = r0 + b.ny * b.pitch;
      const float* r3 = r2 + b.pitch;
      const float tz = ps.t3, ty = ps.t2, tx = ps.t1;
      const float sz = 1.0f - tz, sy = 1.0f - ty, sx = 1.0f - tx;
      const float c00 = r0[0] * sz + r0[1] * tz;
      const float c01 = r1[0] * sz + r1[1] * tz;
      const float c10 = r2[0] * sz + r2[1] * tz;
      const float c11 = r3[0] * sz + r3[1] * tz;
      const float c0 = c00 * sy + c01 * ty;
      const float c1 = c10 * sy + c11 * ty;
      o = c0 * sx + c1 * tx;
    }
    epi((i * d.n2 + j) * d.n3 + k, o);
  }
}

inline dim3 sweep_grid(const Dims& d, const Tile& T, int nplanes) {
  const int ntk = (d.n3 + T.tk - 1) / T.tk, ntj = (d.n2 + T.tj - 1) / T.tj;
  return dim3(ntk * ntj, nplanes, 1);
}

}  // namespace stg
}  // namespace vr

namespace vr {
namespace stg {

// ---- warp-tiled, double-buffered staged sweep ---------------------------------
// Each WARP owns a stream of tiles (32 consecutive x3 voxels x WR x2 rows of
// one x1 plane) and keeps the NEXT tile's source box in flight while it
// gathers the current one: per warp two box buffers and two mbarriers, box
// bounds from warp reductions, one cp.async.bulk per box row issued by the
// warp's own lanes -- no CTA-wide barrier anywhere, so a warp never waits for
// another warp's copy.  (The CTA-tiled kernel above spends ~1/3 of its stall
// samples in the mbarrier wait for its single box.)  Taps and arithmetic are
// the CTA kernel's, so results equal the direct gather's to the ulp.
// MEASURED SLOWER on B200 (C2 advect 0.550 vs 0.293 ms, incremental step 0.617
// vs 0.342): a 32-voxel-wide box row is a ~160-B bulk copy, 3.5x more copy
// requests per byte than the CTA tile's ~560-B rows, and 8 KB double buffers
// leave 12 warps / SM.  Kept behind vr_set_gather_mode(5) as the record.
constexpr int WR = 2;          // x2 rows per warp tile (points per lane)
constexpr int WCAP = 2048;     // floats per box buffer (8 KB)
constexpr int WWARPS = 4;      // warps per CTA

struct WBox {
  int x0, y0, s, nx, ny, len, pitch, ok;
};

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int ORDER, bool SLAB, class Epi>
__global__ void __launch_bounds__(WWARPS * 32, 3) wsweep_kernel(PlaneSrc<1, SLAB> src, Dims d,
                                                               const float* __restrict__ disp, int x0, int nx,
                                                               Epi epi) {
  constexpr int LO = ORDER == ORDER_CUBIC ? 1 : 0;
  constexpr int HI = ORDER == ORDER_CUBIC ? 2 : 1;
  extern __shared__ __align__(128) float wbox[];
  __shared__ __align__(8) unsigned long long bars[WWARPS][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* buf0 = wbox + (size_t)(w * 2) * WCAP;
  float* buf1 = buf0 + WCAP;
  const unsigned bar0 = smem_u32(&bars[w][0]), bar1 = smem_u32(&bars[w][1]);
  if (lane == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar1, 1);
  }
  __syncwarp();
  const int64_t N = d.n();
  const int psz = d.n2 * d.n3;
  const int tk = d.n3 >> 5, tj = d.n2 / WR;
  const int64_t ntiles = (int64_t)nx * tj * tk;
  const int64_t stride = (int64_t)gridDim.x * WWARPS;
  int64_t t = (int64_t)blockIdx.x * WWARPS + w;

  // per-tile lane state
  auto tile_pos = [&](int64_t tt, int& i, int& j0, int& k) {
    const int kb = (int)(tt % tk);
    const int64_t r = tt / tk;
    const int jb = (int)(r % tj);
    i = (int)(r / tj) + x0;
    j0 = jb * WR;
    k = kb * 32 + lane;
  };
  auto load_disp = [&](int64_t tt, float (&dv)[3][WR]) {
    int i, j0, k;
    tile_pos(tt, i, j0, k);
#pragma unroll
    for (int p = 0; p < WR; ++p) {
      const int id = (i * d.n2 + j0 + p) * d.n3 + k;
      dv[0][p] = __ldg(disp + id);
      dv[1][p] = __ldg(disp + N + id);
      dv[2][p] = __ldg(disp + 2 * N + id);
    }
  };
  // box of a tile (uniform across the warp) and the copies into `buf` on `bar`
  auto make_box = [&](int64_t tt, const float (&dv)[3][WR]) -> WBox {
    int i, j0, k;
    tile_pos(tt, i, j0, k);
    int mn1 = INT_MAX, mx1 = INT_MIN, mn2 = INT_MAX, mx2 = INT_MIN, mn3 = INT_MAX, mx3 = INT_MIN;
    bool bad = false;
#pragma unroll
    for (int p = 0; p < WR; ++p) {
      const PointSplit<ORDER, SLAB> ps(src, d, i, j0 + p, k, dv[0][p], dv[1][p], dv[2][p]);
      bad |= ps.bad;
      mn1 = min(mn1, ps.b1); mx1 = max(mx1, ps.b1);
      mn2 = min(mn2, ps.b2); mx2 = max(mx2, ps.b2);
      mn3 = min(mn3, ps.b3); mx3 = max(mx3, ps.b3);
    }
    WBox b;
    mn1 = __reduce_min_sync(~0u, mn1); mx1 = __reduce_max_sync(~0u, mx1);
    mn2 = __reduce_min_sync(~0u, mn2); mx2 = __reduce_max_sync(~0u, mx2);
    mn3 = __reduce_min_sync(~0u, mn3); mx3 = __reduce_max_sync(~0u, mx3);
    const bool anybad = __any_sync(~0u, bad);
    b.x0 = mn1 - LO;
    b.nx = mx1 - mn1 + LO + HI + 1;
    b.y0 = mn2 - LO;
    b.ny = mx2 - mn2 + LO + HI + 1;
    b.s = floor4(mn3 - LO);
    b.len = ((mx3 + HI + 1 - b.s) + 3) & ~3;
    b.pitch = (b.len & 31) == 0 ? b.len + 4 : b.len;
    b.ok = !anybad && b.len <= d.n3 && b.ny <= d.n2 && (SLAB || b.nx <= d.n1) && b.nx * b.ny <= 64 &&
           b.nx * b.ny * b.pitch <= WCAP;
    return b;
  };
  auto issue = [&](const WBox& b, float* buf, unsigned bar) {
    if (!b.ok) return;
    __syncwarp();
    fence_proxy_async();   // the warp's earlier generic reads of `buf` before the async-proxy writes
    if (lane == 0) mbar_expect_tx(bar, (unsigned)(b.nx * b.ny * b.len * 4));
    __syncwarp();
    int s = b.s % d.n3;
    if (s < 0) s += d.n3;
    const int first = min(b.len, d.n3 - s);
    const int nrows = b.nx * b.ny;
    for (int r = lane; r < nrows; r += 32) {
      const int xr = r / b.ny, yr = r - xr * b.ny;
      int x = b.x0 + xr;
      if (!SLAB) x = wrap1(x, d.n1);
      int y = (b.y0 + yr) % d.n2;
      if (y < 0) y += d.n2;
      const float* row = src.plane(0, x, psz) + y * d.n3;
      const unsigned dst = smem_u32(buf + r * b.pitch);
      bulk_g2s(dst, row + s, (unsigned)first * 4u, bar);
      if (first < b.len) bulk_g2s(dst + first * 4u, row, (unsigned)(b.len - first) * 4u, bar);
    }
  };

  float dv[3][WR];
  WBox box;
  unsigned ph0 = 0, ph1 = 0;
  if (t < ntiles) {
    load_disp(t, dv);
    box = make_box(t, dv);
    issue(box, buf0, bar0);
  }
  for (int it = 0; t < ntiles; ++it, t += stride) {
    const bool odd = it & 1;
    float* cur = odd ? buf1 : buf0;
    float* nxt = odd ? buf0 : buf1;
    const unsigned cbar = odd ? bar1 : bar0, nbar = odd ? bar0 : bar1;
    // prefetch the next tile's displacements and box
    const int64_t t2 = t + stride;
    float dv2[3][WR];
    WBox box2;
    box2.ok = 0;
    if (t2 < ntiles) {
      load_disp(t2, dv2);
      box2 = make_box(t2, dv2);
      issue(box2, nxt, nbar);
    }
    int i, j0, k;
    tile_pos(t, i, j0, k);
    if (box.ok) {
      mbar_wait(cbar, odd ? ph1 : ph0);
      if (odd) ph1 ^= 1u; else ph0 ^= 1u;
#pragma unroll
      for (int p = 0; p < WR; ++p) {
        const int j = j0 + p;
        const PointSplit<ORDER, SLAB> ps(src, d, i, j, k, dv[0][p], dv[1][p], dv[2][p]);
        float o;
        if (ORDER == ORDER_CUBIC) {
          float wx[4], wy[4], wz[4];
          lagrange4(ps.t1, wx);
          lagrange4(ps.t2, wy);
          lagrange4(ps.t3, wz);
          const int xs = box.ny * box.pitch;
          const float* base = cur + ((ps.b1 - 1 - box.x0) * box.ny + (ps.b2 - 1 - box.y0)) * box.pitch +
                              (ps.b3 - 1 - box.s);
          float acc = 0.0f;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            float sa = 0.0f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float* r = base + a * xs + c * box.pitch;
              const float sb = wz[0] * r[0] + wz[1] * r[1] + wz[2] * r[2] + wz[3] * r[3];
              sa += wy[c] * sb;
            }
            acc += wx[a] * sa;
          }
          o = acc;
        } else {
          const float* r0 = cur + ((ps.b1 - box.x0) * box.ny + (ps.b2 - box.y0)) * box.pitch + (ps.b3 - box.s);
          const float* r1 = r0 + box.pitch;
          const float* r2 = r0 + box.ny * box.pitch;
          const float* r3 = r2 + box.pitch;
          const float tz = ps.t3, ty = ps.t2, tx = ps.t1;
          const float sz = 1.0f - tz, sy = 1.0f - ty, sx = 1.0f - tx;
          const float c00 = r0[0] * sz + r0[1] * tz;
          const float c01 = r1[0] * sz + r1[1] * tz;
          const float c10 = r2[0] * sz + r2[1] * tz;
          const float c11 = r3[0] * sz + r3[1] * tz;
          const float c0 = c00 * sy + c01 * ty;
          const float c1 = c10 * sy + c11 * ty;
          o = c0 * sx + c1 * tx;
        }
        epi((i * d.n2 + j) * d.n3 + k, o);
      }
    } else {   // box over budget / non-finite displacement: direct gather (same taps and order)
#pragma unroll 1
      for (int p = 0; p < WR; ++p) {
        const int j = j0 + p;
        float o;
        gather_disp_lean<ORDER, 1, SLAB>(src, d, i, j, k, dv[0][p], dv[1][p], dv[2][p], &o);
        epi((i * d.n2 + j) * d.n3 + k, o);
      }
    }
#pragma unroll
    for (int p = 0; p < WR; ++p) {
      dv[0][p] = dv2[0][p];
      dv[1][p] = dv2[1][p];
      dv[2][p] = dv2[2][p];
    }
    box = box2;
  }
}

inline bool wsweep_ok(const Dims& d) { return d.n3 % 32 == 0 && d.n2 % WR == 0; }

}  // namespace stg
}  // namespace vr
