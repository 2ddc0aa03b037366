// Semi-Lagrangian transport kernels: scattered interpolation, RK2 trace,
// trapezoidal source factors, and the state / adjoint / incremental-state /
// Jacobian sweeps of /root/reference/pkg/src/velreg/transport.py.
//
// Characteristics are stored as DISPLACEMENTS in index units (12 B/voxel):
// departure point of voxel (i,j,k) = (i-d1, j-d2, k-d3).  The reference stores
// absolute radians wrapped to [0,2pi) (transport.py:75); both describe the same
// point, the displacement keeps full fp32 precision for the interpolation
// fraction at any grid size.
#include <algorithm>
#include "common.cuh"
#include "interp.cuh"
#include "stage_tma.cuh"
#include "../../include/velreg_b200.h"

namespace vr {

__device__ __forceinline__ void voxel_ijk(int idx, const Dims& d, int& i, int& j, int& k) {
  k = idx % d.n3;
  int r = idx / d.n3;
  j = r % d.n2;
  i = r / d.n2;
}

// 3-D launch: x = x3 (TPB threads), y = x2, z = x1 -- no index divisions
struct Vox {
  int i, j, k, idx;
  bool ok;
};
__device__ __forceinline__ Vox vox3(const Dims& d, int x0 = 0) {
  Vox v;
  v.k = blockIdx.x * blockDim.x + threadIdx.x;
  v.j = blockIdx.y;
  v.i = blockIdx.z + x0;   // x0: first x1 plane of a partial (interior / boundary) launch
  v.ok = v.k < d.n3;
  v.idx = (v.i * d.n2 + v.j) * d.n3 + v.k;
  return v;
}
inline int vox_tpb(const Dims& d) { return d.n3 >= 128 ? 128 : ((d.n3 + 31) / 32) * 32; }
inline dim3 vox_grid(const Dims& d, int nplanes = -1) {
  return dim3((d.n3 + vox_tpb(d) - 1) / vox_tpb(d), d.n2, nplanes < 0 ? d.n1 : nplanes);
}

__device__ __forceinline__ void flag_nonfinite(int* flag, float v) {
  if (flag && !isfinite(v)) atomicOr(flag, 1);
}

// ---- interpolate_values at absolute points in radians (interp.py:112-128) ----
template <int ORDER, typename PT>
__global__ void __launch_bounds__(256) interp_points_kernel(const float* __restrict__ src, Dims d,
                                                            const PT* __restrict__ pts, int64_t npts,
                                                            double h1, double h2, double h3,
                                                            float* __restrict__ out) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  // index = p / h (interp.py:23-25), floor, fraction; computed in f64
  double q1 = (double)pts[p] / h1, q2 = (double)pts[npts + p] / h2, q3 = (double)pts[2 * npts + p] / h3;
  double f1 = floor(q1), f2 = floor(q2), f3 = floor(q3);
  // base index into [0,n) (a full modulo only off the principal period), then
  // the lean gather: one row pointer per stencil row, immediate-offset taps
  int ix = (int)f1, iy = (int)f2, iz = (int)f3;
  if ((unsigned)ix >= (unsigned)d.n1) ix = wrap_idx(ix, d.n1);
  if ((unsigned)iy >= (unsigned)d.n2) iy = wrap_idx(iy, d.n2);
  if ((unsigned)iz >= (unsigned)d.n3) iz = wrap_idx(iz, d.n3);
  const PlaneSrc<1, false> s{src, nullptr, nullptr, d.n(), 0, 0, d.n1};
  float o;
  gather_lean<ORDER, 1, false>(s, d, ix, iy, iz, (float)(q1 - f1), (float)(q2 - f2), (float)(q3 - f3), &o);
  out[p] = o;
}

// ---- RK2 (Heun) trace, both directions, optional source factors -------------
// transport.py:66-76 (trace), :94-110 (TransportOperators factors):
//   x* = x - dt v(x);  X = x - dt/2 (v(x) + v(x*))           (forward)
//   backward trace is the same with -v (transport.py:102)
//   jac = (1 + dt/2 div(X_f)) / (1 - dt/2 div(x)),  adj likewise with X_b
// Uses the general flat-index gather (its 3-component form keeps register
// pressure low; the trace runs once per velocity iterate).  SLAB: v and div are
// contiguous ghost-extended slabs of L1 + 2w planes (component stride Ne); the
// departure x1 index is shifted by w and clamped instead of wrapped.
template <int ORDER, bool SLAB>
__device__ __forceinline__ void trace_gather(const float* const* p, const Dims& ds, int w, int i, int j, int k,
                                             float d1, float d2, float d3, float* out, int nc) {
  int ix, iy, iz;
  float tx, ty, tz;
  split_coord(i, d1, ix, tx);
  split_coord(j, d2, iy, ty);
  split_coord(k, d3, iz, tz);
  if (SLAB) ix = clampi(ix + w, 1, ds.n1 - 3);
  SrcF32 s{{p[0], p[nc > 1 ? 1 : 0], p[nc > 2 ? 2 : 0]}, 0};
  if (nc == 3)
    gather<ORDER, 3>(s, ds, ix, iy, iz, tx, ty, tz, out);
  else
    gather<ORDER, 1>(s, ds, ix, iy, iz, tx, ty, tz, out);
}

template <int ORDER, bool FACTORS, bool SLAB>
__global__ void __launch_bounds__(256) trace_kernel(const float* __restrict__ v, Dims d, int w, float dt, float ih1,
                                                    float ih2, float ih3, float* __restrict__ disp_f,
                                                    float* __restrict__ disp_b, const float* __restrict__ div,
                                                    float* __restrict__ fac_f, float* __restrict__ fac_b) {
  const int64_t N = d.n();
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N) return;
  int i, j, k;
  voxel_ijk(idx, d, i, j, k);
  const Dims ds{SLAB ? d.n1 + 2 * w : d.n1, d.n2, d.n3};   // source dims
  const int64_t Ne = ds.n();
  const int sidx = SLAB ? idx + w * d.n2 * d.n3 : idx;    // own voxel in the source
  const float v1 = __ldg(v + sidx), v2 = __ldg(v + Ne + sidx), v3 = __ldg(v + 2 * Ne + sidx);
  const float a1 = dt * v1 * ih1, a2 = dt * v2 * ih2, a3 = dt * v3 * ih3;
  const float* sv[3] = {v, v + Ne, v + 2 * Ne};
  float vs[3];
  const float half = 0.5f * dt;
  // forward: x* = x - dt v
  trace_gather<ORDER, SLAB>(sv, ds, w, i, j, k, a1, a2, a3, vs, 3);
  const float f1 = half * (v1 + vs[0]) * ih1, f2 = half * (v2 + vs[1]) * ih2, f3 = half * (v3 + vs[2]) * ih3;
  disp_f[idx] = f1;
  disp_f[N + idx] = f2;
  disp_f[2 * N + idx] = f3;
  // backward: x* = x + dt v, X = x + dt/2 (v + v(x*))
  trace_gather<ORDER, SLAB>(sv, ds, w, i, j, k, -a1, -a2, -a3, vs, 3);
  const float b1 = -half * (v1 + vs[0]) * ih1, b2 = -half * (v2 + vs[1]) * ih2, b3 = -half * (v3 + vs[2]) * ih3;
  disp_b[idx] = b1;
  disp_b[N + idx] = b2;
  disp_b[2 * N + idx] = b3;
  if (FACTORS) {
    const float* sd[1] = {div};
    const float denom = 1.0f - half * __ldg(div + sidx);
    float dv;
    trace_gather<ORDER, SLAB>(sd, ds, w, i, j, k, f1, f2, f3, &dv, 1);
    fac_f[idx] = (1.0f + half * dv) / denom;
    trace_gather<ORDER, SLAB>(sd, ds, w, i, j, k, b1, b2, b3, &dv, 1);
    fac_b[idx] = (1.0f + half * dv) / denom;
  }
}

// v (3, N) SoA -> (N) float4 AoS (v1, v2, v3, 0) for the trace's velocity gathers
__global__ void __launch_bounds__(256) soa_to_aos4_kernel(const float* __restrict__ v, int64_t N,
                                                          float4* __restrict__ q) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) q[i] = make_float4(__ldg(v + i), __ldg(v + N + i), __ldg(v + 2 * N + i), 0.0f);
}

// trace_kernel's arithmetic with the velocity gathers from the float4 copy
// (SLAB: vq is the ghost-extended slab, L1 + 2w planes, x1 clamped as in trace_gather)
template <int ORDER, bool FACTORS, bool SLAB>
__global__ void __launch_bounds__(256) trace_aos_kernel(const float4* __restrict__ vq, Dims d, int w, float dt,
                                                        float ih1, float ih2, float ih3, float* __restrict__ disp_f,
                                                        float* __restrict__ disp_b, const float* __restrict__ div,
                                                        float* __restrict__ fac_f, float* __restrict__ fac_b) {
  const int64_t N = d.n();
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N) return;
  int i, j, k;
  voxel_ijk(idx, d, i, j, k);
  const Dims ds{SLAB ? d.n1 + 2 * w : d.n1, d.n2, d.n3};   // source dims
  const int sidx = SLAB ? idx + w * d.n2 * d.n3 : idx;    // own voxel in the source
  const float4 vv = __ldg(vq + sidx);
  const float v1 = vv.x, v2 = vv.y, v3 = vv.z;
  const float a1 = dt * v1 * ih1, a2 = dt * v2 * ih2, a3 = dt * v3 * ih3;
  const SrcAoS4 sq{vq};
  float vs[3];
  const float half = 0.5f * dt;
  int ix, iy, iz;
  float tx, ty, tz;
  split_coord(i, a1, ix, tx);
  split_coord(j, a2, iy, ty);
  split_coord(k, a3, iz, tz);
  if (SLAB) ix = clampi(ix + w, 1, ds.n1 - 3);
  gather_aos3<ORDER>(sq, ds, ix, iy, iz, tx, ty, tz, vs);
  const float f1 = half * (v1 + vs[0]) * ih1, f2 = half * (v2 + vs[1]) * ih2, f3 = half * (v3 + vs[2]) * ih3;
  disp_f[idx] = f1;
  disp_f[N + idx] = f2;
  disp_f[2 * N + idx] = f3;
  split_coord(i, -a1, ix, tx);
  split_coord(j, -a2, iy, ty);
  split_coord(k, -a3, iz, tz);
  if (SLAB) ix = clampi(ix + w, 1, ds.n1 - 3);
  gather_aos3<ORDER>(sq, ds, ix, iy, iz, tx, ty, tz, vs);
  const float b1 = -half * (v1 + vs[0]) * ih1, b2 = -half * (v2 + vs[1]) * ih2, b3 = -half * (v3 + vs[2]) * ih3;
  disp_b[idx] = b1;
  disp_b[N + idx] = b2;
  disp_b[2 * N + idx] = b3;
  if (FACTORS) {
    const float* sd[1] = {div};
    const float denom = 1.0f - half * __ldg(div + sidx);
    float dv;
    trace_gather<ORDER, SLAB>(sd, ds, w, i, j, k, f1, f2, f3, &dv, 1);
    fac_f[idx] = (1.0f + half * dv) / denom;
    trace_gather<ORDER, SLAB>(sd, ds, w, i, j, k, b1, b2, b3, &dv, 1);
    fac_b[idx] = (1.0f + half * dv) / denom;
  }
}

// Periodic single-domain trace on the lean gather (3-D launch, no index
// divisions, one conditional wrap per axis, immediate-offset x3 taps): the same
// Heun steps and factors as trace_kernel, 3 components gathered per tap row.
template <int ORDER, bool FACTORS>
__global__ void __launch_bounds__(128, 5) trace_lean_kernel(const float* __restrict__ v, Dims d, float dt, float ih1,
                                                         float ih2, float ih3, float* __restrict__ disp_f,
                                                         float* __restrict__ disp_b, const float* __restrict__ div,
                                                         float* __restrict__ fac_f, float* __restrict__ fac_b) {
  const Vox p = vox3(d);
  if (!p.ok) return;
  const int64_t N = d.n();
  const PlaneSrc<3, false> sv{v, nullptr, nullptr, N, 0, 0, d.n1};
  const float v1 = __ldg(v + p.idx), v2 = __ldg(v + N + p.idx), v3 = __ldg(v + 2 * N + p.idx);
  const float a1 = dt * v1 * ih1, a2 = dt * v2 * ih2, a3 = dt * v3 * ih3;
  const float half = 0.5f * dt;
  float vs[3];
  gather_disp_lean<ORDER, 3, false>(sv, d, p.i, p.j, p.k, a1, a2, a3, vs);
  const float f1 = half * (v1 + vs[0]) * ih1, f2 = half * (v2 + vs[1]) * ih2, f3 = half * (v3 + vs[2]) * ih3;
  disp_f[p.idx] = f1;
  disp_f[N + p.idx] = f2;
  disp_f[2 * N + p.idx] = f3;
  gather_disp_lean<ORDER, 3, false>(sv, d, p.i, p.j, p.k, -a1, -a2, -a3, vs);
  const float b1 = -half * (v1 + vs[0]) * ih1, b2 = -half * (v2 + vs[1]) * ih2, b3 = -half * (v3 + vs[2]) * ih3;
  disp_b[p.idx] = b1;
  disp_b[N + p.idx] = b2;
  disp_b[2 * N + p.idx] = b3;
  if (FACTORS) {
    const PlaneSrc<1, false> sd{div, nullptr, nullptr, N, 0, 0, d.n1};
    const float denom = 1.0f - half * __ldg(div + p.idx);
    float dv;
    gather_disp_lean<ORDER, 1, false>(sd, d, p.i, p.j, p.k, f1, f2, f3, &dv);
    fac_f[p.idx] = (1.0f + half * dv) / denom;
    gather_disp_lean<ORDER, 1, false>(sd, d, p.i, p.j, p.k, b1, b2, b3, &dv);
    fac_b[p.idx] = (1.0f + half * dv) / denom;
  }
}

// 0 (default): tricubic velocity gathers from a float4 (AoS) copy of v, one 16-B
// load per tap (C2 trace + FD8 div 2.69 -> 2.38 ms; trilinear unchanged at
// 0.79 ms, so it keeps the SoA gathers); 2: general flat-index trace on the
// SoA field (round-1 default); 1: lean
// periodic trace -- measured SLOWER on B200 (C2 cubic 3.83 vs 2.41 ms per
// trace).  Same arithmetic in all three; vr_set_trace_mode selects for A/B.
static int g_trace_mode = 0;

// ---- one semi-Lagrangian step: dst = interp(src, X) [* factor] --------------
// state  : transport.py:130-133 (no factor)
// adjoint: transport.py:154-155 (factor = adj_numer/adj_denom, backward trace)
// jacobian: transport.py:194-195 (factor = jac_numer/jac_denom)
template <int ORDER, bool SCALE, bool SLAB>
__global__ void __launch_bounds__(128) advect_kernel(PlaneSrc<1, SLAB> src, Dims d, const float* __restrict__ disp,
                                                     const float* __restrict__ fac, float* __restrict__ dst,
                                                     int* flag, int x0) {
  const int64_t N = d.n();
  const Vox p = vox3(d, x0);
  if (!p.ok) return;
  const int idx = p.idx;
  float o;
  gather_disp_lean<ORDER, 1, SLAB>(src, d, p.i, p.j, p.k, __ldg(disp + idx), __ldg(disp + N + idx),
                                   __ldg(disp + 2 * N + idx), &o);
  if (SCALE) o *= __ldg(fac + idx);
  dst[idx] = o;
  flag_nonfinite(flag, o);
}

// ---- incremental state (transport.py:160-185) --------------------------------
// s_j = -(vt . grad m^j);  u_0 = dt/2 s_0
// m~_{j+1} = interp(u_j, X_f) + dt/2 s_{j+1};  u_{j+1} = m~_{j+1} + dt/2 s_{j+1}
__device__ __forceinline__ float inc_source(const float* __restrict__ vt, const float* __restrict__ g, int64_t N,
                                            int idx) {
  return -(__ldg(vt + idx) * __ldg(g + idx) + __ldg(vt + N + idx) * __ldg(g + N + idx) +
           __ldg(vt + 2 * N + idx) * __ldg(g + 2 * N + idx));
}

__global__ void __launch_bounds__(256) incstate_init_kernel(const float* __restrict__ vt,
                                                            const float* __restrict__ g0, int64_t N, float half,
                                                            float* __restrict__ u0) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N) return;
  u0[idx] = half * inc_source(vt, g0, N, idx);
}

template <int ORDER, bool SLAB>
__global__ void __launch_bounds__(128) incstate_step_kernel(PlaneSrc<1, SLAB> u, Dims d,
                                                            const float* __restrict__ disp,
                                                            const float* __restrict__ vt,
                                                            const float* __restrict__ gnext, float half,
                                                            int last, float* __restrict__ out, int* flag, int x0) {
  const int64_t N = d.n();
  const Vox p = vox3(d, x0);
  if (!p.ok) return;
  const int idx = p.idx;
  float o;
  gather_disp_lean<ORDER, 1, SLAB>(u, d, p.i, p.j, p.k, __ldg(disp + idx), __ldg(disp + N + idx),
                                   __ldg(disp + 2 * N + idx), &o);
  const float hs = half * inc_source(vt, gnext, N, idx);
  float m = o + hs;
  if (last == 0) m = m + hs;
  else if (last == 2) m = -m;
  out[idx] = m;
  flag_nonfinite(flag, m);
}

// ---- staged sweeps (stage_tma.cuh): epilogues of the advect / incstate steps ----
template <bool SCALE>
struct AdvectEpi {
  const float* __restrict__ fac;
  float* __restrict__ dst;
  int* flag;
  __device__ __forceinline__ void operator()(int idx, float o) const {
    if (SCALE) o *= __ldg(fac + idx);
    dst[idx] = o;
    flag_nonfinite(flag, o);
  }
};

struct IncEpi {
  const float* __restrict__ vt;
  const float* __restrict__ gnext;
  int64_t N;
  float half;
  int last;
  float* __restrict__ out;
  int* flag;
  __device__ __forceinline__ void operator()(int idx, float o) const {
    const float hs = half * inc_source(vt, gnext, N, idx);
    float m = o + hs;
    if (last == 0) m = m + hs;
    else if (last == 2) m = -m;
    out[idx] = m;
    flag_nonfinite(flag, m);
  }
};

// ---- trapezoidal body force (optim.py:162-171) --------------------------------
// b = sum_j w_j lam^j grad m^j, w = dt/2 at j in {0,n}, dt otherwise; f64 accumulator
__global__ void __launch_bounds__(256) body_force_kernel(const float* __restrict__ lam,
                                                         const float* __restrict__ gm, int nt, int64_t N,
                                                         double dt, float* __restrict__ out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int j = 0; j <= nt; ++j) {
    const double w = (j == 0 || j == nt) ? 0.5 * dt : dt;
    const float wl = (float)(w * (double)__ldg(lam + (int64_t)j * N + idx));
    const float* g = gm + (int64_t)j * 3 * N;
    a0 += (double)(wl * __ldg(g + idx));
    a1 += (double)(wl * __ldg(g + N + idx));
    a2 += (double)(wl * __ldg(g + 2 * N + idx));
  }
  out[idx] = (float)a0;
  out[N + idx] = (float)a1;
  out[2 * N + idx] = (float)a2;
}

// One trapezoid term of the body force with the f64 accumulator kept in HBM
// (lean layout: grad m^j recomputed per term instead of stored as a series).
// The per-voxel arithmetic and summation order are body_force_kernel's, so the
// result is bit-identical:  acc (+)= (double)(RN(w*(double)lam) * g);  on the
// last term out = (float)acc.  mode: 0 = first term (acc =), 1 = middle,
// 2 = last (acc += then write out).
__global__ void __launch_bounds__(256) body_force_term_kernel(const float* __restrict__ lam,
                                                              const float* __restrict__ g, int64_t N, double w,
                                                              int mode, double* __restrict__ acc,
                                                              float* __restrict__ out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N) return;
  const float wl = (float)(w * (double)__ldg(lam + idx));
  double a0 = (double)(wl * __ldg(g + idx));
  double a1 = (double)(wl * __ldg(g + N + idx));
  double a2 = (double)(wl * __ldg(g + 2 * N + idx));
  const double z0 = mode != 0 ? acc[idx] : 0.0;          // 0.0 + x keeps body_force_kernel's zero signs
  const double z1 = mode != 0 ? acc[N + idx] : 0.0;
  const double z2 = mode != 0 ? acc[2 * N + idx] : 0.0;
  a0 = z0 + a0;
  a1 = z1 + a1;
  a2 = z2 + a2;
  if (mode == 2) {
    out[idx] = (float)a0;
    out[N + idx] = (float)a1;
    out[2 * N + idx] = (float)a2;
  } else {
    acc[idx] = a0;
    acc[N + idx] = a1;
    acc[2 * N + idx] = a2;
  }
}

// ---- label transport (synth.py:121-131) ---------------------------------------
// First step gathers the indicator of `id` straight from the label map; the last
// step thresholds at 0.5 and writes `id` (labels processed in ascending order, so
// overlaps resolve to the larger id as in the reference).
template <int ORDER, bool FROM_LABELS, bool TO_LABELS, bool SLAB>
__global__ void __launch_bounds__(128) label_step_kernel(PlaneSrc<1, SLAB> src, const int* __restrict__ lab_in,
                                                         int id, Dims d, const float* __restrict__ disp,
                                                         float* __restrict__ dst, int* __restrict__ lab_out,
                                                         int x0) {
  const int64_t N = d.n();
  const Vox p = vox3(d, x0);
  if (!p.ok) return;
  const int i = p.i, j = p.j, k = p.k, idx = p.idx;
  float o;
  const float d1 = __ldg(disp + idx), d2 = __ldg(disp + N + idx), d3 = __ldg(disp + 2 * N + idx);
  if (FROM_LABELS) {
    SrcLabel s{lab_in, id};
    gather_disp<ORDER, 1>(s, d, i, j, k, d1, d2, d3, &o);
  } else {
    gather_disp_lean<ORDER, 1, SLAB>(src, d, i, j, k, d1, d2, d3, &o);
  }
  if (TO_LABELS) {
    if (o >= 0.5f) lab_out[idx] = id;
  } else {
    dst[idx] = o;
  }
}

template <int NC>
PlaneSrc<NC, true> slab_src(const float* mid, const float* lo, const float* hi, int64_t mid_cs, int64_t ghost_cs,
                            int w, int L1) {
  return PlaneSrc<NC, true>{mid, lo, hi, mid_cs, ghost_cs, w, L1};
}

template <int NC>
PlaneSrc<NC, false> full_src(const float* mid, int64_t cs) {
  return PlaneSrc<NC, false>{mid, mid, mid, cs, cs, 0, 0};
}

// ---- displacement -> absolute points in radians (Characteristics.points) ----
__global__ void disp_to_points_kernel(const float* __restrict__ disp, Dims d, double* __restrict__ pts) {
  const int64_t N = d.n();
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N) return;
  int ijk[3];
  voxel_ijk(idx, d, ijk[0], ijk[1], ijk[2]);
  const int n[3] = {d.n1, d.n2, d.n3};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double q = (double)ijk[a] - (double)disp[a * N + idx];
    double h = kTwoPi / n[a];
    double x = q * h;
    x = fmod(x, kTwoPi);
    if (x < 0) x += kTwoPi;
    pts[a * N + idx] = x;
  }
}

}  // namespace vr

using namespace vr;

#define VR_DISPATCH_ORDER(order, ...)                     \
  if ((order) == 1) {                                     \
    constexpr int ORD = ORDER_LINEAR;                     \
    __VA_ARGS__;                                          \
  } else if ((order) == 3) {                              \
    constexpr int ORD = ORDER_CUBIC;                      \
    __VA_ARGS__;                                          \
  } else {                                                \
    return VR_ERR_ARG;                                    \
  }

extern "C" {

int vr_interp_points(const float* src, const int64_t dims[3], const void* pts, int pts_is_f64, int64_t npts,
                     int order, float* out, void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (npts < 0 || !src || !out || (!pts && npts)) return VR_ERR_ARG;
  if (npts == 0) return VR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const double h1 = kTwoPi / d.n1, h2 = kTwoPi / d.n2, h3 = kTwoPi / d.n3;
  unsigned g = grid_for(npts, 256);
  VR_DISPATCH_ORDER(order, {
    if (pts_is_f64)
      interp_points_kernel<ORD, double><<<g, 256, 0, s>>>(src, d, (const double*)pts, npts, h1, h2, h3, out);
    else
      interp_points_kernel<ORD, float><<<g, 256, 0, s>>>(src, d, (const float*)pts, npts, h1, h2, h3, out);
  });
  VR_CHECK_LAUNCH();
  return VR_OK;
}

}  // extern "C"

// Slab arguments: lo/hi == nullptr -> periodic single-domain call; otherwise the
// source is the local slab (L1 = dims[0] planes) with w ghost planes in lo / hi.
struct SlabArgs {
  const float* lo;
  const float* hi;
  int w;
  bool on() const { return lo != nullptr; }
};

// Stream-ordered scratch (cudaMallocAsync) stays in the device's default pool
// between calls instead of being returned to the OS at every synchronisation
// (release threshold 0 by default: a 268 MB re-allocation per trace).
static void keep_pool_memory() {
  static thread_local int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

static int trace_impl(const float* v, const int64_t dims[3], int64_t n1_global, int w, const float* div, double dt,
                      int order, float* disp_fwd, float* disp_bwd, float* fac_jac, float* fac_adj, void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!v || !disp_fwd || !disp_bwd || !(dt > 0)) return VR_ERR_ARG;
  const bool factors = div != nullptr;
  if (factors && (!fac_jac || !fac_adj)) return VR_ERR_ARG;
  const bool slab = w >= 0;
  if (slab && (w < 2 || w > d.n1)) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const float ih1 = (float)(n1_global / kTwoPi), ih2 = (float)(d.n2 / kTwoPi), ih3 = (float)(d.n3 / kTwoPi);
  const unsigned g = grid_for(d.n(), 256);
  VR_DISPATCH_ORDER(order, {
    if (g_trace_mode == 0 && ORD == ORDER_CUBIC) {
      // tricubic velocity gathers from a float4 copy (v1, v2, v3, 0) of v (or
      // of the ghost-extended slab): one 16-B load per tap (trilinear measured
      // equal and keeps the SoA gathers)
      const int64_t Ne = slab ? (int64_t)(d.n1 + 2 * w) * d.n2 * d.n3 : d.n();
      float4* vq = nullptr;
      keep_pool_memory();
      if (cudaMallocAsync((void**)&vq, sizeof(float4) * Ne, s) != cudaSuccess) return VR_ERR_ALLOC;
      soa_to_aos4_kernel<<<grid_for(Ne, 256), 256, 0, s>>>(v, Ne, vq);
      const int ww = slab ? w : 0;
      if (slab && factors)
        trace_aos_kernel<ORD, true, true><<<g, 256, 0, s>>>(vq, d, ww, (float)dt, ih1, ih2, ih3, disp_fwd, disp_bwd,
                                                            div, fac_jac, fac_adj);
      else if (slab)
        trace_aos_kernel<ORD, false, true><<<g, 256, 0, s>>>(vq, d, ww, (float)dt, ih1, ih2, ih3, disp_fwd,
                                                             disp_bwd, nullptr, nullptr, nullptr);
      else if (factors)
        trace_aos_kernel<ORD, true, false><<<g, 256, 0, s>>>(vq, d, 0, (float)dt, ih1, ih2, ih3, disp_fwd, disp_bwd,
                                                             div, fac_jac, fac_adj);
      else
        trace_aos_kernel<ORD, false, false><<<g, 256, 0, s>>>(vq, d, 0, (float)dt, ih1, ih2, ih3, disp_fwd,
                                                              disp_bwd, nullptr, nullptr, nullptr);
      cudaFreeAsync(vq, s);
    } else if (slab && factors)
      trace_kernel<ORD, true, true><<<g, 256, 0, s>>>(v, d, w, (float)dt, ih1, ih2, ih3, disp_fwd, disp_bwd, div,
                                                      fac_jac, fac_adj);
    else if (slab)
      trace_kernel<ORD, false, true><<<g, 256, 0, s>>>(v, d, w, (float)dt, ih1, ih2, ih3, disp_fwd, disp_bwd,
                                                       nullptr, nullptr, nullptr);
    else if (g_trace_mode == 1 && factors)
      trace_lean_kernel<ORD, true><<<vox_grid(d), vox_tpb(d), 0, s>>>(v, d, (float)dt, ih1, ih2, ih3, disp_fwd,
                                                                       disp_bwd, div, fac_jac, fac_adj);
    else if (g_trace_mode == 1)
      trace_lean_kernel<ORD, false><<<vox_grid(d), vox_tpb(d), 0, s>>>(v, d, (float)dt, ih1, ih2, ih3, disp_fwd,
                                                                        disp_bwd, nullptr, nullptr, nullptr);
    else if (factors)
      trace_kernel<ORD, true, false><<<g, 256, 0, s>>>(v, d, 0, (float)dt, ih1, ih2, ih3, disp_fwd, disp_bwd, div,
                                                       fac_jac, fac_adj);
    else
      trace_kernel<ORD, false, false><<<g, 256, 0, s>>>(v, d, 0, (float)dt, ih1, ih2, ih3, disp_fwd, disp_bwd,
                                                        nullptr, nullptr, nullptr);
  });
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// Staged sweeps (stage_tma.cuh) for rows of a multiple of 32 voxels;
// vr_set_gather_mode(0) selects the direct per-point kernels (A/B checks).
static int g_gather_mode = 1;
// Cubic only: the trilinear sweep (8 taps, 2.7 TB/s direct) measured slower staged.
// cp.async.bulk needs 16-byte-aligned global rows: the row offsets are
// multiples of 128 B (n3 % 32 == 0, x3 start a multiple of 4 floats), so the
// field base pointers decide; anything less aligned takes the direct gather.
static bool use_staged(int order, const Dims& d, const float* src, const float* lo = nullptr,
                       const float* hi = nullptr) {
  const uintptr_t a = (uintptr_t)src | (uintptr_t)lo | (uintptr_t)hi;
  return g_gather_mode >= 1 && order == ORDER_CUBIC && stg::staged_ok(d) && (a & 15) == 0;
}

template <int ORD, bool SLAB, class Epi, class CF>
static void launch_staged_cfg(const PlaneSrc<1, SLAB>& ps, const Dims& d, const float* disp, int x0, int nx, Epi epi,
                              cudaStream_t s) {
  const stg::Tile T = stg::tile_for(d, CF::PPT);
  stg::sweep_kernel<ORD, SLAB, Epi, CF><<<stg::sweep_grid(d, T, nx), stg::NT, CF::kSmemBudget, s>>>(ps, d, disp, T,
                                                                                                 x0, epi);
}

template <int ORD, bool SLAB, class Epi>
static void launch_wsweep(const PlaneSrc<1, SLAB>& ps, const Dims& d, const float* disp, int x0, int nx, Epi epi,
                          cudaStream_t s) {
  const size_t sm = sizeof(float) * stg::WCAP * 2 * stg::WWARPS;
  static int slots = 0;
  if (!slots) {
    cudaFuncSetAttribute(stg::wsweep_kernel<ORD, SLAB, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, stg::wsweep_kernel<ORD, SLAB, Epi>, stg::WWARPS * 32, sm);
    slots = sms * (per > 0 ? per : 1);
  }
  const int64_t ntiles = (int64_t)nx * (d.n2 / stg::WR) * (d.n3 / 32);
  const int64_t need = (ntiles + stg::WWARPS - 1) / stg::WWARPS;
  const unsigned grid = (unsigned)std::min<int64_t>(need, slots);
  stg::wsweep_kernel<ORD, SLAB, Epi><<<grid, stg::WWARPS * 32, sm, s>>>(ps, d, disp, x0, nx, epi);
}

template <int ORD, bool SLAB, class Epi>
static void launch_staged(const PlaneSrc<1, SLAB>& ps, const Dims& d, const float* disp, int x0, int nx, Epi epi,
                          cudaStream_t s) {
  if (g_gather_mode == 5 && stg::wsweep_ok(d)) {
    launch_wsweep<ORD, SLAB, Epi>(ps, d, disp, x0, nx, epi, s);
    return;
  }
  if (g_gather_mode == 2) launch_staged_cfg<ORD, SLAB, Epi, stg::CfgB>(ps, d, disp, x0, nx, epi, s);
  else if (g_gather_mode == 3) launch_staged_cfg<ORD, SLAB, Epi, stg::CfgC>(ps, d, disp, x0, nx, epi, s);
  else if (g_gather_mode == 4) launch_staged_cfg<ORD, SLAB, Epi, stg::CfgD>(ps, d, disp, x0, nx, epi, s);
  else launch_staged_cfg<ORD, SLAB, Epi, stg::CfgA>(ps, d, disp, x0, nx, epi, s);
}

static int advect_impl(const float* src, SlabArgs sg, const int64_t dims[3], const float* disp, const float* factor,
                       int order, float* dst, int* nonfinite_flag, void* stream, int x0 = 0, int nx = -1) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!src || !disp || !dst || src == dst) return VR_ERR_ARG;
  if (sg.on() && (sg.w < 1 || sg.w > d.n1 || !sg.hi)) return VR_ERR_ARG;
  if (nx < 0) nx = d.n1;
  if (x0 < 0 || nx < 0 || x0 + nx > d.n1) return VR_ERR_ARG;
  if (nx == 0) return VR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (use_staged(order, d, src, sg.lo, sg.hi)) {
    VR_DISPATCH_ORDER(order, {
      if (sg.on()) {
        auto ps = slab_src<1>(src, sg.lo, sg.hi, 0, 0, sg.w, d.n1);
        if (factor)
          launch_staged<ORD>(ps, d, disp, x0, nx, AdvectEpi<true>{factor, dst, nonfinite_flag}, s);
        else
          launch_staged<ORD>(ps, d, disp, x0, nx, AdvectEpi<false>{nullptr, dst, nonfinite_flag}, s);
      } else {
        auto ps = full_src<1>(src, 0);
        if (factor)
          launch_staged<ORD>(ps, d, disp, x0, nx, AdvectEpi<true>{factor, dst, nonfinite_flag}, s);
        else
          launch_staged<ORD>(ps, d, disp, x0, nx, AdvectEpi<false>{nullptr, dst, nonfinite_flag}, s);
      }
    });
    VR_CHECK_LAUNCH();
    return VR_OK;
  }
  const dim3 g = vox_grid(d, nx);
  const int tpb = vox_tpb(d);
  VR_DISPATCH_ORDER(order, {
    if (sg.on()) {
      auto ps = slab_src<1>(src, sg.lo, sg.hi, 0, 0, sg.w, d.n1);
      if (factor)
        advect_kernel<ORD, true, true><<<g, tpb, 0, s>>>(ps, d, disp, factor, dst, nonfinite_flag, x0);
      else
        advect_kernel<ORD, false, true><<<g, tpb, 0, s>>>(ps, d, disp, nullptr, dst, nonfinite_flag, x0);
    } else {
      auto ps = full_src<1>(src, 0);
      if (factor)
        advect_kernel<ORD, true, false><<<g, tpb, 0, s>>>(ps, d, disp, factor, dst, nonfinite_flag, x0);
      else
        advect_kernel<ORD, false, false><<<g, tpb, 0, s>>>(ps, d, disp, nullptr, dst, nonfinite_flag, x0);
    }
  });
  VR_CHECK_LAUNCH();
  return VR_OK;
}

static int incstate_impl(const float* u, SlabArgs sg, const int64_t dims[3], const float* disp_fwd, const float* vt,
                         const float* gradm_next, double dt, int order, int last, float* out, int* nonfinite_flag,
                         void* stream, int x0 = 0, int nx = -1) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!u || !disp_fwd || !vt || !gradm_next || !out || u == out) return VR_ERR_ARG;
  if (sg.on() && (sg.w < 1 || sg.w > d.n1 || !sg.hi)) return VR_ERR_ARG;
  if (nx < 0) nx = d.n1;
  if (x0 < 0 || nx < 0 || x0 + nx > d.n1) return VR_ERR_ARG;
  if (nx == 0) return VR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (use_staged(order, d, u, sg.lo, sg.hi)) {
    const IncEpi epi{vt, gradm_next, d.n(), (float)(0.5 * dt), last, out, nonfinite_flag};
    VR_DISPATCH_ORDER(order, {
      if (sg.on())
        launch_staged<ORD>(slab_src<1>(u, sg.lo, sg.hi, 0, 0, sg.w, d.n1), d, disp_fwd, x0, nx, epi, s);
      else
        launch_staged<ORD>(full_src<1>(u, 0), d, disp_fwd, x0, nx, epi, s);
    });
    VR_CHECK_LAUNCH();
    return VR_OK;
  }
  const dim3 g = vox_grid(d, nx);
  const int tpb = vox_tpb(d);
  VR_DISPATCH_ORDER(order, {
    if (sg.on())
      incstate_step_kernel<ORD, true><<<g, tpb, 0, s>>>(slab_src<1>(u, sg.lo, sg.hi, 0, 0, sg.w, d.n1), d, disp_fwd,
                                                        vt, gradm_next, (float)(0.5 * dt), last, out, nonfinite_flag, x0);
    else
      incstate_step_kernel<ORD, false><<<g, tpb, 0, s>>>(full_src<1>(u, 0), d, disp_fwd, vt, gradm_next,
                                                         (float)(0.5 * dt), last, out, nonfinite_flag, x0);
  });
  VR_CHECK_LAUNCH();
  return VR_OK;
}

extern "C" {

int vr_trace_rk2(const float* v, const int64_t dims[3], double dt, int order, float* disp_fwd, float* disp_bwd,
                 const float* div, float* fac_jac, float* fac_adj, void* stream) {
  if (!dims) return VR_ERR_ARG;
  return trace_impl(v, dims, dims[0], -1, div, dt, order, disp_fwd, disp_bwd, fac_jac, fac_adj, stream);
}

int vr_trace_rk2_slab(const float* v_ext, const int64_t dims[3], int64_t n1_global, int w, double dt, int order,
                      float* disp_fwd, float* disp_bwd, const float* div_ext, float* fac_jac, float* fac_adj,
                      void* stream) {
  if (w < 0) return VR_ERR_ARG;
  return trace_impl(v_ext, dims, n1_global, w, div_ext, dt, order, disp_fwd, disp_bwd, fac_jac, fac_adj, stream);
}

int vr_advect(const float* src, const int64_t dims[3], const float* disp, const float* factor, int order,
              float* dst, int* nonfinite_flag, void* stream) {
  return advect_impl(src, SlabArgs{nullptr, nullptr, 0}, dims, disp, factor, order, dst, nonfinite_flag, stream);
}

int vr_advect_slab(const float* src, const float* src_lo, const float* src_hi, const int64_t dims[3], int w,
                   const float* disp, const float* factor, int order, float* dst, int* nonfinite_flag, int x_begin,
                   int x_count, void* stream) {
  if (!src_lo || !src_hi) return VR_ERR_ARG;
  return advect_impl(src, SlabArgs{src_lo, src_hi, w}, dims, disp, factor, order, dst, nonfinite_flag, stream,
                     x_begin, x_count);
}

int vr_incstate_init(const float* vt, const float* gradm0, const int64_t dims[3], double dt, float* u0,
                     void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!vt || !gradm0 || !u0) return VR_ERR_ARG;
  incstate_init_kernel<<<grid_for(d.n(), 256), 256, 0, (cudaStream_t)stream>>>(vt, gradm0, d.n(),
                                                                               (float)(0.5 * dt), u0);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_incstate_step(const float* u, const int64_t dims[3], const float* disp_fwd, const float* vt,
                     const float* gradm_next, double dt, int order, int last, float* out, int* nonfinite_flag,
                     void* stream) {
  return incstate_impl(u, SlabArgs{nullptr, nullptr, 0}, dims, disp_fwd, vt, gradm_next, dt, order, last, out,
                       nonfinite_flag, stream);
}

int vr_incstate_step_slab(const float* u, const float* u_lo, const float* u_hi, const int64_t dims[3], int w,
                          const float* disp_fwd, const float* vt, const float* gradm_next, double dt, int order,
                          int last, float* out, int* nonfinite_flag, int x_begin, int x_count, void* stream) {
  if (!u_lo || !u_hi) return VR_ERR_ARG;
  return incstate_impl(u, SlabArgs{u_lo, u_hi, w}, dims, disp_fwd, vt, gradm_next, dt, order, last, out,
                       nonfinite_flag, stream, x_begin, x_count);
}

int vr_body_force(const float* lam_series, const float* gradm_series, int n_t, const int64_t dims[3], double dt,
                  float* out, void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!lam_series || !gradm_series || !out || n_t < 1) return VR_ERR_ARG;
  body_force_kernel<<<grid_for(d.n(), 256), 256, 0, (cudaStream_t)stream>>>(lam_series, gradm_series, n_t, d.n(),
                                                                            dt, out);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_body_force_term(const float* lam, const float* gradm, const int64_t dims[3], double weight, int mode,
                       double* acc, float* out, void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!lam || !gradm || !acc || mode < 0 || mode > 2 || (mode == 2 && !out)) return VR_ERR_ARG;
  body_force_term_kernel<<<grid_for(d.n(), 256), 256, 0, (cudaStream_t)stream>>>(lam, gradm, d.n(), weight, mode,
                                                                                 acc, out);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_label_step(const float* src, const int* labels_in, int label_id, const int64_t dims[3], const float* disp,
                  int order, float* dst, int* labels_out, void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!disp || (!src && !labels_in) || (!dst && !labels_out)) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 g = vox_grid(d);
  const int tpb = vox_tpb(d);
  const bool from_l = labels_in != nullptr, to_l = labels_out != nullptr;
  auto ps = full_src<1>(src ? src : reinterpret_cast<const float*>(labels_in), 0);
  VR_DISPATCH_ORDER(order, {
    if (from_l && to_l)
      label_step_kernel<ORD, true, true, false><<<g, tpb, 0, s>>>(ps, labels_in, label_id, d, disp, nullptr,
                                                                  labels_out, 0);
    else if (from_l)
      label_step_kernel<ORD, true, false, false><<<g, tpb, 0, s>>>(ps, labels_in, label_id, d, disp, dst, nullptr, 0);
    else if (to_l)
      label_step_kernel<ORD, false, true, false><<<g, tpb, 0, s>>>(ps, nullptr, label_id, d, disp, nullptr,
                                                                   labels_out, 0);
    else
      label_step_kernel<ORD, false, false, false><<<g, tpb, 0, s>>>(ps, nullptr, label_id, d, disp, dst, nullptr, 0);
  });
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// slab label step from a float indicator / advected field with ghost blocks
int vr_label_step_slab(const float* src, const float* src_lo, const float* src_hi, int label_id,
                       const int64_t dims[3], int w, const float* disp, int order, float* dst, int* labels_out,
                       void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!src || !src_lo || !src_hi || !disp || w < 1 || w > d.n1 || (!dst && !labels_out)) return VR_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 g = vox_grid(d);
  const int tpb = vox_tpb(d);
  auto ps = slab_src<1>(src, src_lo, src_hi, 0, 0, w, d.n1);
  VR_DISPATCH_ORDER(order, {
    if (labels_out)
      label_step_kernel<ORD, false, true, true><<<g, tpb, 0, s>>>(ps, nullptr, label_id, d, disp, nullptr,
                                                                  labels_out, 0);
    else
      label_step_kernel<ORD, false, false, true><<<g, tpb, 0, s>>>(ps, nullptr, label_id, d, disp, dst, nullptr, 0);
  });
  VR_CHECK_LAUNCH();
  return VR_OK;
}

int vr_set_gather_mode(int mode) {
  const int prev = g_gather_mode;
  g_gather_mode = mode;
  return prev;
}

int vr_set_trace_mode(int mode) {
  const int prev = g_trace_mode;
  g_trace_mode = mode;
  return prev;
}

int vr_disp_to_points(const float* disp, const int64_t dims[3], double* pts, void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!disp || !pts) return VR_ERR_ARG;
  disp_to_points_kernel<<<grid_for(d.n(), 256), 256, 0, (cudaStream_t)stream>>>(disp, d, pts);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

}  // extern "C"
