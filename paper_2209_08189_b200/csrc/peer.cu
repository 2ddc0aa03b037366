// Peer-memory transport between the GPUs of one node (one process per GPU).
//
// The x1-slab decomposition (dist.py) moves data between ranks at three kinds
// of points: ghost planes for the stencils, the spectral transposes, and
// scalar reductions.  The first two run here over NVLink / NVSwitch without
// NCCL kernels:
//   * symmetric buffers: cudaMalloc'd receive buffers whose CUDA IPC handles
//     every rank opens, so a rank can store straight into a peer's buffer;
//   * ghost planes: one SM put kernel (halo_put_kernel) storing both faces
//     into the neighbours' IPC-mapped ghost blocks -- measured ~12 us cheaper
//     per exchange than a pair of copy-engine copies (vr_peer_copy stays for
//     the bulk all-to-all blocks);
//   * transposes: the spectral pack / x1 kernels store their output tiles
//     directly into the destination rank's receive buffer (spectral.cu,
//     vr_dspec_*_peer) -- the transpose IS the kernel's epilogue;
//   * completion: per (source, channel) uint64 epoch flags in the receiver's
//     memory, written by the sender after its data (a one-thread release-store
//     kernel ordered behind the copy / producer kernel, system-scope fence
//     first) and awaited on the receiver's stream with cuStreamWaitValue64
//     (no spinning kernel, no host round trip).
// Epochs only grow, so flags are never reset; a receive buffer is reused only
// after a later exchange with the same peer has completed.
#include <cuda.h>
#include <cstring>
#include <algorithm>
#include <mutex>
#include "common.cuh"
#include "../../include/velreg_b200.h"

namespace {

typedef CUresult (*PFN_waitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_batchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

PFN_waitValue64 g_wait = nullptr;
PFN_batchMemOp g_batch = nullptr;
std::once_flag g_once;

void load_driver_entry_points() {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait = reinterpret_cast<PFN_waitValue64>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_batch = reinterpret_cast<PFN_batchMemOp>(fn);
  });
}

constexpr int kMaxFlags = 8;
struct FlagSet {
  unsigned long long* f[kMaxFlags];
  int n;
};

// one-thread release store of an epoch into a (peer) flag, after a
// system-scope fence: everything this stream wrote before is visible first
__global__ void signal_kernel(unsigned long long* flag, unsigned long long value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

// the same for up to kMaxFlags flags in one launch (one per destination rank)
__global__ void signal_many_kernel(FlagSet fs, unsigned long long value) {
  __threadfence_system();
#pragma unroll
  for (int i = 0; i < kMaxFlags; ++i)
    if (i < fs.n) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fs.f[i]), "l"(value) : "memory");
}

// Ghost-plane put: the first w planes of every component go to the left
// neighbour's hi ghost block, the last w planes to the right neighbour's lo
// block (both IPC-mapped), one float4 per thread per step.  An SM copy: a
// copy-engine copy of these 1-3 MB blocks costs ~12 us of launch latency each.
__global__ void __launch_bounds__(256) halo_put_kernel(const float4* __restrict__ src, int ncomp, int64_t cstride4,
                                                       int64_t plane4, int L1, int w, float4* __restrict__ left_hi,
                                                       float4* __restrict__ right_lo) {
  const int64_t blk4 = (int64_t)w * plane4;          // float4s per component block
  const int64_t n = 2 * ncomp * blk4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t side = e / (ncomp * blk4), r = e - side * ncomp * blk4;
    const int64_t c = r / blk4, o = r - c * blk4;
    if (side == 0) left_hi[c * blk4 + o] = src[c * cstride4 + o];
    else right_lo[c * blk4 + o] = src[c * cstride4 + (int64_t)(L1 - w) * plane4 + o];
  }
}

}  // namespace

extern "C" {

// ghost planes of a (ncomp, L1, N2, N3) float slab into the neighbours' blocks
// (ncomp, w, N2, N3); plane = N2 * N3 (a multiple of 4), 16-byte-aligned pointers
int vr_peer_halo_put(const float* src, int ncomp, int L1, int64_t plane, int w, float* left_hi, float* right_lo,
                     void* stream) {
  if (!src || !left_hi || !right_lo || ncomp < 1 || w < 1 || w > L1 || plane % 4) return VR_ERR_ARG;
  if (((uintptr_t)src | (uintptr_t)left_hi | (uintptr_t)right_lo) & 15) return VR_ERR_ARG;
  const int64_t n4 = 2 * (int64_t)ncomp * w * (plane / 4);
  const unsigned grid = (unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
  halo_put_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(src), ncomp, (int64_t)L1 * plane / 4, plane / 4, L1, w,
      reinterpret_cast<float4*>(left_hi), reinterpret_cast<float4*>(right_lo));
  VR_CHECK_LAUNCH();
  return VR_OK;
}


int vr_peer_malloc(int64_t bytes, void** ptr, void* handle_out) {
  if (bytes <= 0 || !ptr || !handle_out) return VR_ERR_ARG;
  void* p = nullptr;
  if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) return VR_ERR_ALLOC;
  if (cudaMemset(p, 0, (size_t)bytes) != cudaSuccess ||
      cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle_out), p) != cudaSuccess) {
    cudaFree(p);
    return VR_ERR_ALLOC;
  }
  *ptr = p;
  return VR_OK;
}

int vr_peer_free(void* ptr) {
  if (ptr) cudaFree(ptr);
  return VR_OK;
}

int vr_peer_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return VR_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return VR_ERR_ALLOC;
  *ptr = p;
  return VR_OK;
}

int vr_peer_close(void* ptr) {
  if (ptr) cudaIpcCloseMemHandle(ptr);
  return VR_OK;
}

int vr_peer_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// device-to-device copy on the copy engines (the destination may be a peer's
// IPC-mapped buffer)
int vr_peer_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes && (!dst || !src))) return VR_ERR_ARG;
  if (!bytes) return VR_OK;
  if (cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) != cudaSuccess)
    return VR_ERR_LAUNCH;
  return VR_OK;
}

// flag := value, ordered after all prior work of `stream` (flag may be a peer's)
int vr_peer_signal(unsigned long long* flag, unsigned long long value, void* stream) {
  if (!flag) return VR_ERR_ARG;
  signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// flags[0..n) := value in one launch, ordered after all prior work of `stream`
int vr_peer_signal_many(unsigned long long* const* flags, int n, unsigned long long value, void* stream) {
  if (!flags || n < 1 || n > kMaxFlags) return VR_ERR_ARG;
  FlagSet fs{};
  for (int i = 0; i < n; ++i) {
    if (!flags[i]) return VR_ERR_ARG;
    fs.f[i] = flags[i];
  }
  fs.n = n;
  signal_many_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(fs, value);
  VR_CHECK_LAUNCH();
  return VR_OK;
}

// `stream` waits until every *flags[i] >= value: one batched stream memory
// operation (cuStreamBatchMemOp) instead of n separate waits
int vr_peer_wait_many(const unsigned long long* const* flags, int n, unsigned long long value, void* stream) {
  if (!flags || n < 1 || n > kMaxFlags) return VR_ERR_ARG;
  load_driver_entry_points();
  if (!g_batch) {
    for (int i = 0; i < n; ++i)
      if (int rc = vr_peer_wait(flags[i], value, stream)) return rc;
    return VR_OK;
  }
  CUstreamBatchMemOpParams ops[kMaxFlags];
  memset(ops, 0, sizeof(ops));
  for (int i = 0; i < n; ++i) {
    if (!flags[i]) return VR_ERR_ARG;
    ops[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
    ops[i].waitValue.address = (CUdeviceptr)flags[i];
    ops[i].waitValue.value64 = (cuuint64_t)value;
    ops[i].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
  }
  const CUresult r = g_batch((CUstream)stream, (unsigned)n, ops, 0);
  return r == CUDA_SUCCESS ? VR_OK : VR_ERR_LAUNCH;
}

// `stream` waits until *flag >= value (flag in this GPU's memory)
int vr_peer_wait(const unsigned long long* flag, unsigned long long value, void* stream) {
  if (!flag) return VR_ERR_ARG;
  load_driver_entry_points();
  if (!g_wait) return VR_ERR_UNSUPPORTED;
  const CUresult r = g_wait((CUstream)stream, (CUdeviceptr)flag, (cuuint64_t)value, CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? VR_OK : VR_ERR_LAUNCH;
}

}  // extern "C"
