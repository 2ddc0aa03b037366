// Exhaustive check of the FD8 reciprocal division (csrc/fd8.cu div_fast)
// against IEEE division for every float32 bit pattern and every grid spacing
// h = fp32(2*pi/n), n in [lo, hi] (even n; the reference grid's dims are even).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rdc tools/recip_div_check.cu && /tmp/rdc 10 4096
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ float div_fast(float x, float h, float r) {
  const float q = __fmul_rn(x, r);
  const float e = __fmaf_rn(-q, h, x);
  return __fmaf_rn(e, r, q);
}

// counts: [0] mismatches with finite x and finite IEEE quotient, [1] other mismatches
__global__ void check(float h, float r, unsigned long long* counts, unsigned* first) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long bad_fin = 0, bad_other = 0;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < (1ull << 32); u += stride) {
    const float x = __uint_as_float((unsigned)u);
    if (x != x) continue;  // NaN payloads
    const float a = div_fast(x, h, r), b = __fdiv_rn(x, h);
    if (__float_as_uint(a) != __float_as_uint(b)) {
      const bool fin = isfinite(x) && isfinite(b);
      if (fin) {
        ++bad_fin;
        const unsigned ab = (unsigned)u & 0x7fffffffu;
        if (ab < 0x3f800000u) atomicMax(first, ab);        // largest failing |x| below 1
        else atomicMin(first + 1, ab);                     // smallest failing |x| above 1
      }
      else ++bad_other;
    }
  }
  if (bad_fin) atomicAdd(counts, bad_fin);
  if (bad_other) atomicAdd(counts + 1, bad_other);
}

int main(int argc, char** argv) {
  const int lo = argc > 1 ? atoi(argv[1]) : 10, hi = argc > 2 ? atoi(argv[2]) : 4096;
  unsigned long long* c;
  unsigned* first;
  cudaMalloc(&c, 16);
  cudaMalloc(&first, 8);
  unsigned long long tot_fin = 0, tot_other = 0;
  int nbad = 0;
  unsigned lo_max = 0, hi_min = 0xffffffffu;
  for (int n = lo; n <= hi; n += 2) {
    const float h = (float)(6.283185307179586476925286766559 / n);
    const float r = 1.0f / h;
    cudaMemset(c, 0, 16);
    const unsigned init[2] = {0u, 0xffffffffu};
    cudaMemcpy(first, init, 8, cudaMemcpyHostToDevice);
    check<<<148 * 16, 256>>>(h, r, c, first);
    unsigned long long hc[2];
    unsigned hf[2];
    cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(hf, first, 8, cudaMemcpyDeviceToHost);
    tot_fin += hc[0];
    tot_other += hc[1];
    lo_max = hf[0] > lo_max ? hf[0] : lo_max;
    hi_min = hf[1] < hi_min ? hf[1] : hi_min;
    if (hc[0] && nbad++ < 5) {
      printf("n=%d h=%a: %llu finite mismatches, largest small |x| %a, smallest large |x| %a\n", n, h, hc[0],
             __builtin_bit_cast(float, hf[0]), __builtin_bit_cast(float, hf[1]));
    }
  }
  printf("n in [%d,%d]: finite mismatches %llu (all with |x| <= %a or >= %a), non-finite mismatches %llu, err=%s\n",
         lo, hi, tot_fin, __builtin_bit_cast(float, lo_max), __builtin_bit_cast(float, hi_min), tot_other,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
