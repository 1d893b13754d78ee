// Microbenchmarks that pick the counting design for the n-gram passes on B200:
// streaming read bandwidth, shared / distributed-shared / L2 atomic throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_stream(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <int MODE>  // 0 atomicOr w/ ret, 1 atomicAdd no ret, 2 plain store, 3 load
__global__ void k_smem(int iters, uint32_t words_mask, uint32_t* out) {
  extern __shared__ uint32_t s[];
  for (uint32_t i = threadIdx.x; i <= words_mask; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t x = mix(blockIdx.x * blockDim.x + threadIdx.x);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t h = mix(x);
    uint32_t w = h & words_mask;
    if (MODE == 0) acc += atomicOr(&s[w], 1u << (h >> 27));
    else if (MODE == 1) atomicAdd(&s[w], 1u);
    else if (MODE == 2) s[w] = h;
    else acc += s[w];
  }
  __syncthreads();
  if (acc == 0x12345678 || s[threadIdx.x] == 0x87654321) out[0] = acc;
}

template <int MODE>  // 0 red u32, 1 red u64, 2 atom u32 ret, 3 atomicOr ret u32, 4 hot-skewed red u32
__global__ void k_gmem(int iters, uint32_t mask, void* tab, uint32_t* out) {
  uint32_t x = mix(blockIdx.x * blockDim.x + threadIdx.x);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t h = mix(x);
    uint32_t w = h & mask;
    if (MODE == 0) atomicAdd((uint32_t*)tab + w, 1u);
    else if (MODE == 1) atomicAdd((unsigned long long*)tab + w, 1ull);
    else if (MODE == 2) acc += atomicAdd((uint32_t*)tab + w, 1u);
    else if (MODE == 3) acc += atomicOr((uint32_t*)tab + (w >> 5), 1u << (h & 31));
    else if (MODE == 4) { if ((h >> 28) == 0) w &= 15; atomicAdd((uint32_t*)tab + w, 1u); }
  }
  if (acc == 0x12345678) out[0] = acc;
}

// Distributed shared memory: each CTA of a cluster owns words_mask+1 words; ops go to
// the CTA selected by the top bits of the hash.
template <int CS>
__global__ void k_dsmem(int iters, uint32_t words_mask, uint32_t* out) {
  extern __shared__ uint32_t s[];
  cg::cluster_group cl = cg::this_cluster();
  for (uint32_t i = threadIdx.x; i <= words_mask; i += blockDim.x) s[i] = 0;
  cl.sync();
  uint32_t x = mix(blockIdx.x * blockDim.x + threadIdx.x);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t h = mix(x);
    uint32_t w = h & words_mask;
    uint32_t r = (h >> 24) % CS;
    uint32_t* rs = cl.map_shared_rank(s, r);
    acc += atomicOr(rs + w, 1u << (h >> 27));
  }
  cl.sync();
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  printf("device %s sms %d l2 %d MB smem/block optin %zu clock %d kHz\n", prop.name, sms, prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin, prop.clockRate);
  uint32_t* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float ms;

  // A: streaming read
  {
    size_t bytes = 4ull << 30; void* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 1, bytes));
    for (int blocksPerSm : {2, 4, 8}) {
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(a));
        k_stream<<<sms * blocksPerSm, 512>>>((const uint4*)p, bytes / 16, out);
        CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      }
      printf("stream_read bps=%d: %.1f GB/s\n", blocksPerSm, bytes / ms / 1e6);
    }
    CK(cudaFree(p));
  }
  // B: shared-memory ops
  {
    const int iters = 4096;
    for (int kb : {32, 64, 128, 200}) {
      uint32_t words = (kb * 1024) / 4; uint32_t mask = 1; while (mask * 2 <= words) mask *= 2; mask -= 1;
      size_t sm = (mask + 1) * 4;
      CK(cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      CK(cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      CK(cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      CK(cudaFuncSetAttribute(k_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      for (int threads : {512, 1024}) {
        int blocks = sms * (kb <= 64 ? 2 : 1);
        double ops = (double)blocks * threads * iters;
        const char* names[4] = {"atomicOr_ret", "atomicAdd", "store", "load"};
        for (int mode = 0; mode < 4; ++mode) {
          for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(a));
            if (mode == 0) k_smem<0><<<blocks, threads, sm>>>(iters, mask, out);
            if (mode == 1) k_smem<1><<<blocks, threads, sm>>>(iters, mask, out);
            if (mode == 2) k_smem<2><<<blocks, threads, sm>>>(iters, mask, out);
            if (mode == 3) k_smem<3><<<blocks, threads, sm>>>(iters, mask, out);
            CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
          }
          CK(cudaGetLastError());
          printf("smem %s %dKB thr=%d blocks=%d: %.1f Gop/s (%.2f op/clk/SM)\n", names[mode], kb, threads, blocks, ops / ms / 1e6,
                 ops / (ms * 1e-3) / sms / (prop.clockRate * 1e3));
        }
      }
    }
  }
  // C: global atomics
  {
    const int iters = 256;
    void* tab; CK(cudaMalloc(&tab, 1ull << 30)); CK(cudaMemset(tab, 0, 1ull << 30));
    const char* names[5] = {"red_u32", "red_u64", "atom_u32_ret", "atomicOr_ret_bitmap", "red_u32_hot"};
    for (uint32_t mb : {4u, 64u, 128u, 512u}) {
      for (int mode = 0; mode < 5; ++mode) {
        uint32_t elem = (mode == 1) ? 8 : 4;
        uint32_t mask = (uint32_t)(((uint64_t)mb << 20) / elem) - 1;
        if (mode == 3) mask = (uint32_t)(((uint64_t)mb << 20) * 8) - 1;  // bit index
        int blocks = sms * 4, threads = 512;
        double ops = (double)blocks * threads * iters;
        for (int rep = 0; rep < 3; ++rep) {
          CK(cudaEventRecord(a));
          switch (mode) {
            case 0: k_gmem<0><<<blocks, threads>>>(iters, mask, tab, out); break;
            case 1: k_gmem<1><<<blocks, threads>>>(iters, mask, tab, out); break;
            case 2: k_gmem<2><<<blocks, threads>>>(iters, mask, tab, out); break;
            case 3: k_gmem<3><<<blocks, threads>>>(iters, mask, tab, out); break;
            case 4: k_gmem<4><<<blocks, threads>>>(iters, mask, tab, out); break;
          }
          CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
        }
        CK(cudaGetLastError());
        printf("gmem %s %u MB: %.1f Gop/s\n", names[mode], mb, ops / ms / 1e6);
      }
    }
    CK(cudaFree(tab));
  }
  // D: distributed shared memory atomics
  {
    const int iters = 2048;
    auto run = [&](auto kern, int cs, int kb) {
      uint32_t mask = (kb * 1024 / 4) - 1;
      size_t sm = (mask + 1) * 4;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      if (cs > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t cfg = {};
      int blocks = (sms / cs) * cs;
      cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = sm;
      cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr; cfg.numAttrs = 1;
      int ncl = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
      printf("dsmem cs=%d maxActiveClusters=%d (%s)\n", cs, ncl, cudaGetErrorString(e));
      if (ncl <= 0) { cudaGetLastError(); return; }
      cfg.gridDim = dim3(ncl * cs);
      double ops = (double)ncl * cs * 1024 * iters;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(a));
        e = cudaLaunchKernelEx(&cfg, kern, iters, mask, out);
        if (e != cudaSuccess) { printf("launch fail %s\n", cudaGetErrorString(e)); cudaGetLastError(); return; }
        CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      }
      printf("dsmem atomicOr_ret cs=%d %dKB/CTA ctas=%d: %.1f Gop/s\n", cs, kb, ncl * cs, ops / ms / 1e6);
    };
    run(k_dsmem<2>, 2, 128);
    run(k_dsmem<4>, 4, 128);
    run(k_dsmem<8>, 8, 128);
    run(k_dsmem<16>, 16, 128);
  }
  printf("done\n");
  return 0;
}
