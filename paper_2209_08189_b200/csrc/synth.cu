// SYN benchmark template on the device (/root/reference/pkg/src/velreg/synth.py:77-101).
//
// A template is a union of star-shaped regions: shape i (1..n) covers voxel x
// when |u| <= |Y_l^m(theta + theta_i, phi + phi_i)|, u = (x - pi) - c_i, with
// phi the polar angle of u (arccos(u3 / |u|), 0 at the centre) and the
// azimuth entering only through a unit-modulus phase (synth.py:71-73).  The
// label of a voxel is the LARGEST covering index (later shapes overwrite,
// synth.py:99).  One thread per voxel evaluates every shape in f64 with the
// reference's operation sequence (np.arccos / np.cos / the upward associated-
// Legendre recurrence, synth.py:42-62); the per-shape random draws (centres
// and quarter turns from numpy's default_rng) are made on the host so the
// random stream is the reference's.  A 1024^3 SYN template (the paper's K
// studies) is then one launch instead of ~26 GB of host f64
// coordinate arrays.
#include "common.cuh"
#include "../../include/velreg_b200.h"

namespace vr {

struct SynShape {
  double c[3];      // centre offset (radians, about the centred lattice)
  double phi_hat;   // quarter turn added to the polar angle
};

// P_l^m(x), Condon-Shortley phase, upward recurrence (synth.py:42-62)
__device__ __forceinline__ double assoc_legendre(int l, int m, double x, double dfact_m) {
  double pmm = 1.0;
  if (m > 0) {
    const double s = sqrt(fmax(1.0 - x * x, 0.0));
    pmm = ((m & 1) ? -1.0 : 1.0) * dfact_m * pow(s, (double)m);
  }
  if (l == m) return pmm;
  double pm1 = x * (2 * m + 1) * pmm;
  if (l == m + 1) return pm1;
  for (int ll = m + 2; ll <= l; ++ll) {
    const double p = (x * (2 * ll - 1) * pm1 - (ll + m - 1) * pmm) / (ll - m);
    pmm = pm1;
    pm1 = p;
  }
  return pm1;
}

__global__ void __launch_bounds__(256) syn_labels_kernel(Dims d, const SynShape* __restrict__ shapes, int nshapes,
                                                         int l, int m, double norm, double dfact_m,
                                                         double fixed_radius, int x0, int* __restrict__ labels,
                                                         float* __restrict__ image) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d.n3) return;
  const int j = blockIdx.y, il = blockIdx.z, i = il + x0;   // d = global dims; x0 offsets a slab
  // centred coordinates x - pi (grid.py:53-56 lattice i * (2 pi / n), synth.py:87)
  const double x = (double)i * (kTwoPi / d.n1) - 3.14159265358979323846;
  const double y = (double)j * (kTwoPi / d.n2) - 3.14159265358979323846;
  const double z = (double)k * (kTwoPi / d.n3) - 3.14159265358979323846;
  int lab = 0;
  for (int s = 0; s < nshapes; ++s) {
    const SynShape sh = shapes[s];
    const double u0 = x - sh.c[0], u1 = y - sh.c[1], u2 = z - sh.c[2];
    const double r = sqrt(u0 * u0 + u1 * u1 + u2 * u2);   // np.sqrt((u**2).sum(axis=0))
    double radius;
    if (fixed_radius >= 0.0) {
      radius = fixed_radius;
    } else {
      const double cphi = r > 0.0 ? u2 / r : 1.0;
      const double phi = acos(fmin(fmax(cphi, -1.0), 1.0));
      radius = norm * fabs(assoc_legendre(l, m, cos(phi + sh.phi_hat), dfact_m));
    }
    if (r <= radius) lab = s + 1;
  }
  const int64_t idx = ((int64_t)il * d.n2 + j) * d.n3 + k;
  if (labels) labels[idx] = lab;
  if (image) image[idx] = (float)lab;
}

}  // namespace vr

using namespace vr;

extern "C" {

int vr_syn_template(const int64_t dims[3], int x_begin, int x_count, const double* shapes_host, int nshapes, int l,
                    int m, double norm, double dfact_m, double fixed_radius, int* labels, float* image,
                    void* stream) {
  Dims d;
  int rc = dims_from(dims, &d);
  if (rc) return rc;
  if (!shapes_host || nshapes < 1 || nshapes > 4096 || m < 0 || m > l || l > 64) return VR_ERR_ARG;
  if (x_begin < 0 || x_count < 0 || x_begin + x_count > d.n1 || (!labels && !image)) return VR_ERR_ARG;
  if (x_count == 0) return VR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  SynShape* dev = nullptr;
  if (cudaMallocAsync((void**)&dev, sizeof(SynShape) * nshapes, s) != cudaSuccess) return VR_ERR_ALLOC;
  // pageable source: the copy is staged before the call returns
  if (cudaMemcpyAsync(dev, shapes_host, sizeof(SynShape) * nshapes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
    cudaFreeAsync(dev, s);
    return VR_ERR_LAUNCH;
  }
  const dim3 grid((d.n3 + 255) / 256, d.n2, x_count);
  syn_labels_kernel<<<grid, 256, 0, s>>>(d, dev, nshapes, l, m, norm, dfact_m, fixed_radius, x_begin, labels,
                                         image);
  const cudaError_t e = cudaGetLastError();
  cudaFreeAsync(dev, s);
  return e == cudaSuccess ? VR_OK : VR_ERR_LAUNCH;
}

}  // extern "C"
