// select_kernels.cu — canonical top-k of a device count table on sm_100a.
//
// Reference: top_k, proj/src/counting.cpp:52-98 (min-heap over nonzero
// entries, canonical order count desc / gram bytes asc, counting.hpp:38-41;
// returns min(k, nonzero) entries, counting.cpp:72,90-97).
//
// GPU restatement (deterministic, no heap):
//   1. radix-select the k-th largest nonzero count T, MSB digit first (8-bit
//      digits, one histogram pass + one single-block pick per digit).  After
//      the last digit, `need` = how many entries with count == T belong in the
//      answer (#(count > T) = k - need).
//   2. radix-select the need-th smallest gram key Kt among entries with
//      count == T (the tie-break; gram keys are unique per table).
//   3. compact every entry with count > T, or count == T and key <= Kt: exactly
//      min(k, nonzero) entries.
//   4. order them canonically with two stable radix sorts (key asc, then count
//      desc) — CUB DeviceRadixSort, stable by construction.
// Each histogram pass is a streaming read of the table (HBM/L2 bound).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ig_internal.cuh"
#include "kernels.h"

namespace igb {

struct KeyFn {
  const uint64_t* pkeys;  // nullptr: key = id
  uint64_t minv, cmask;   // permuted table index -> id (minv == 0: identity)
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    const uint64_t id = minv ? ((i * minv) & cmask) : i;
    return pkeys ? ((__ldg(pkeys + (id >> 8)) << 8) | (id & 255)) : id;
  }
};

template <typename CT>
__device__ __forceinline__ void load4(const CT* t, uint64_t i, uint64_t c[4]);
template <>
__device__ __forceinline__ void load4<uint32_t>(const uint32_t* t, uint64_t i, uint64_t c[4]) {
  const uint4 v = __ldcs(reinterpret_cast<const uint4*>(t + i));
  c[0] = v.x;
  c[1] = v.y;
  c[2] = v.z;
  c[3] = v.w;
}
template <>
__device__ __forceinline__ void load4<unsigned long long>(const unsigned long long* t, uint64_t i,
                                                          uint64_t c[4]) {
  const ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2*>(t + i));
  const ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2*>(t + i + 2));
  c[0] = a.x;
  c[1] = a.y;
  c[2] = b.x;
  c[3] = b.y;
}

// max count (for the number of digit passes) and the sum of all counts (the
// occurrences the pass counted: the next pass's sparse switch) — per warp,
// then atomicMax / atomicAdd into out[0] / out[1].
template <typename CT>
__global__ void k_max(const CT* __restrict__ t, uint64_t cap4, unsigned long long* out) {
  uint64_t mx = 0, sum = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c[4];
    load4<CT>(t, i * 4, c);
    mx = max(max(mx, c[0]), max(c[1], max(c[2], c[3])));
    sum += c[0] + c[1] + c[2] + c[3];
  }
  for (int d = 16; d; d >>= 1) {
    mx = max(mx, (uint64_t)__shfl_xor_sync(0xffffffffu, mx, d));
    sum += (uint64_t)__shfl_xor_sync(0xffffffffu, sum, d);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, (unsigned long long)mx);
    if (sum) atomicAdd(out + 1, (unsigned long long)sum);
  }
}

// Histogram of digit (v >> shift) & 255 over the entries still in play.
// MODE 0: v = count, entries with count > 0 and high digits == prefix.
// MODE 1: v = key, entries with count == T and high key digits == prefix.
template <typename CT, int MODE>
__global__ void k_hist(const CT* __restrict__ t, uint64_t cap4, KeyFn kf, const SelState* st,
                       int shift, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int hs = shift + 8;
  const uint64_t pre = MODE == 0 ? st->prefix : st->kprefix;
  const uint64_t T = st->T;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c[4];
    load4<CT>(t, i * 4, c);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (MODE == 0) {
        if (c[u] == 0) continue;
        if (hs < 64 && (c[u] >> hs) != (pre >> hs)) continue;
        atomicAdd(&h[(c[u] >> shift) & 255], 1u);
      } else {
        if (c[u] != T) continue;
        const uint64_t key = kf(i * 4 + u);
        if (hs < 64 && (key >> hs) != (pre >> hs)) continue;
        atomicAdd(&h[(key >> shift) & 255], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

// Single block: choose this pass's digit.  MODE 0 scans from the largest
// digit (largest counts), MODE 1 from the smallest (smallest keys).
template <int MODE>
__global__ void k_pick(SelState* st, int shift, int first, uint32_t* hist) {
  if (threadIdx.x == 0) {
    uint64_t r = MODE == 0 ? st->r : st->need;
    if (MODE == 0 && first) {
      uint64_t total = 0;
      for (int d = 0; d < 256; ++d) total += hist[d];
      st->nonzero = total;
      if (total <= r) st->take_all = 1;
    }
    if (!(MODE == 0 && st->take_all)) {
      uint64_t cum = 0;
      for (int i = 0; i < 256; ++i) {
        const int d = MODE == 0 ? 255 - i : i;
        if (cum + hist[d] >= r) {
          if (MODE == 0) st->prefix |= (uint64_t)d << shift;
          else st->kprefix |= (uint64_t)d << shift;
          r -= cum;
          break;
        }
        cum += hist[d];
      }
      if (MODE == 0) st->r = r;
      else st->need = r;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
}

__global__ void k_finish_count_select(SelState* st) {
  if (st->take_all) {
    st->T = 0;  // every nonzero entry is taken
    st->need = 0;
    st->kprefix = ~0ull;
  } else {
    st->T = st->prefix;
    st->need = st->r;
    st->kprefix = 0;
  }
}

// Entries in the answer: count > T, or count == T and key <= Kt.
template <typename CT>
__global__ void k_compact(const CT* __restrict__ t, uint64_t cap4, KeyFn kf, const SelState* st,
                          unsigned long long* __restrict__ n_out, uint64_t* __restrict__ out_keys,
                          uint64_t* __restrict__ out_counts) {
  const uint64_t T = st->T, Kt = st->kprefix;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c[4];
    load4<CT>(t, i * 4, c);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c[u] == 0 || c[u] < T) continue;
      const uint64_t key = kf(i * 4 + u);
      if (c[u] == T && key > Kt) continue;
      const unsigned long long slot = atomicAdd(n_out, 1ull);
      out_keys[slot] = key;
      out_counts[slot] = c[u];
    }
  }
}

__global__ void k_invert(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t n,
                         uint64_t top) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = top - in[i];
}

static int bits_of(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

__global__ void k_set_state(SelState* st, SelState v) { *st = v; }

template <typename CT>
uint64_t select_topk(SelectCtx& x, const CT* table, uint64_t cap, uint64_t k, KeyMap km,
                     int key_bits, uint64_t* out_keys, uint64_t* out_counts) {
  cudaStream_t s = x.stream;
  const uint64_t cap4 = cap / 4;  // cap is a multiple of 4
  // u32 digit histograms and CUB's int item counts bound the table
  if (cap >= 0x7fffffffull)
    throw Error(IG_ECONFIG, "count table of " + std::to_string(cap) +
                                " entries exceeds the selection's 2^31 - 1 limit");
  const KeyFn kf{km.pkeys, km.minv, km.cmask};
  const int threads = 512;
  unsigned blocks = (unsigned)((cap4 + threads - 1) / threads);
  const unsigned maxb = (unsigned)x.num_sms * 4;
  if (blocks > maxb) blocks = maxb;
  if (!blocks) blocks = 1;

  SelState init{};
  init.r = k;
  k_set_state<<<1, 1, 0, s>>>(x.state, init);  // by value: no host copy
  x.launches++;
  IGB_CUDA(cudaMemsetAsync(x.hist, 0, 256 * sizeof(uint32_t), s));
  IGB_CUDA(cudaMemsetAsync(x.scalar, 0, 2 * sizeof(unsigned long long), s));
  k_max<CT><<<blocks, threads, 0, s>>>(table, cap4, x.scalar);
  x.launches++;
  launch_copy(x.h_scalar, x.scalar, 2 * sizeof(unsigned long long), s);  // mapped pinned
  x.launches++;
  IGB_CUDA(cudaStreamSynchronize(s));
  const unsigned long long mx = x.h_scalar[0];
  x.last_sum = x.h_scalar[1];
  if (mx == 0) return 0;  // all-zero table: empty result (counting.cpp:72)
  const int cbits = bits_of(mx);
  const int cpasses = (cbits + 7) / 8;
  for (int p = cpasses - 1; p >= 0; --p) {
    k_hist<CT, 0><<<blocks, threads, 0, s>>>(table, cap4, kf, x.state, p * 8, x.hist);
    k_pick<0><<<1, 256, 0, s>>>(x.state, p * 8, p == cpasses - 1, x.hist);
    x.launches += 2;
  }
  k_finish_count_select<<<1, 1, 0, s>>>(x.state);
  x.launches++;
  launch_copy(x.h_state, x.state, sizeof(SelState), s);
  x.launches++;
  IGB_CUDA(cudaStreamSynchronize(s));
  const SelState hs = *x.h_state;
  if (!hs.take_all) {
    const int kpasses = (key_bits + 7) / 8;
    for (int p = kpasses - 1; p >= 0; --p) {
      k_hist<CT, 1><<<blocks, threads, 0, s>>>(table, cap4, kf, x.state, p * 8, x.hist);
      k_pick<1><<<1, 256, 0, s>>>(x.state, p * 8, 0, x.hist);
      x.launches += 2;
    }
  }
  const uint64_t nsel = hs.take_all ? hs.nonzero : k;
  IGB_CUDA(cudaMemsetAsync(x.scalar, 0, sizeof(unsigned long long), s));
  uint64_t* tk = x.tmp_keys.as<uint64_t>(nsel * 2 + 2);
  uint64_t* tc = x.tmp_counts.as<uint64_t>(nsel * 2 + 2);
  k_compact<CT><<<blocks, threads, 0, s>>>(table, cap4, kf, x.state, x.scalar, tk, tc);
  x.launches++;

  // canonical order: stable sort by key asc, then by count desc
  uint64_t* k2 = tk + nsel;
  uint64_t* c2 = tc + nsel;
  size_t need1 = 0, need2 = 0;
  IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need1, tk, k2, tc, c2, (int)nsel, 0,
                                           key_bits > 0 ? key_bits : 1, s));
  IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need2, tc, out_counts, k2, out_keys,
                                           (int)nsel, 0, cbits > 0 ? cbits : 1, s));
  void* tmp = x.cub_tmp.get(need1 > need2 ? need1 : need2);
  size_t t1 = x.cub_tmp.bytes;
  IGB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t1, tk, k2, tc, c2, (int)nsel, 0,
                                           key_bits > 0 ? key_bits : 1, s));
  // inverted counts so that ascending = count descending
  const uint64_t top = cbits >= 64 ? ~0ull : ((1ull << cbits) - 1);
  unsigned ib = (unsigned)((nsel + 255) / 256);
  if (ib > 4096) ib = 4096;
  if (!ib) ib = 1;
  k_invert<<<ib, 256, 0, s>>>(c2, tc, nsel, top);
  size_t t2 = x.cub_tmp.bytes;
  IGB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t2, tc, c2, k2, out_keys, (int)nsel, 0,
                                           cbits > 0 ? cbits : 1, s));
  k_invert<<<ib, 256, 0, s>>>(c2, out_counts, nsel, top);
  x.launches += 2;  // the two inverts (CUB sort kernels are library launches, not counted)
  IGB_CUDA(cudaGetLastError());
  return nsel;
}

template uint64_t select_topk<uint32_t>(SelectCtx&, const uint32_t*, uint64_t, uint64_t, KeyMap,
                                        int, uint64_t*, uint64_t*);
template uint64_t select_topk<unsigned long long>(SelectCtx&, const unsigned long long*, uint64_t,
                                                  uint64_t, KeyMap, int, uint64_t*, uint64_t*);

}  // namespace igb
