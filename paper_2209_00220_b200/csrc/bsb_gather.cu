// bsb_gather.cu -- locality for row-id gathers.
//
// A lookup of a row-id list in random order (cfg3's unsorted ids) touches one
// random 32-byte sector per slice per id.  Sorting the ids first turns the
// gather into a forward walk over the column (ids that share a block share
// its sectors, and DRAM pages are visited in order); the looked-up values are
// then scattered back to input order.  The host wrappers
// (lookup_*_rows(order="auto")) use this for large unsorted lists.
#include <atomic>
#include <chrono>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>

#include "bsb_common.cuh"

namespace bsb {

constexpr int kBucketBits = 16;

static int gather_grid(int64_t items, int threads) {
  int64_t g = (items + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

__global__ void rows_sample_check_kernel(const int64_t* __restrict__ rows, int64_t n,
                                         unsigned int* __restrict__ bad) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // 0..4095
  const int64_t i = (n - 1) * k / 4096;
  const bool b = i + 1 < n && __ldg(rows + i + 1) < __ldg(rows + i);
  if (__any_sync(kFull, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// keys = row >> shift (the bucket), values = input position
template <typename K>
__global__ void make_pairs_kernel(const int64_t* __restrict__ rows, int64_t n, int shift,
                                  K* __restrict__ keys, K* __restrict__ pos) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (K)(rows[i] >> shift);
    pos[i] = (K)i;
  }
}

template <typename K>
__global__ void unpack_pairs_kernel(const int64_t* __restrict__ rows, const K* __restrict__ pos,
                                    int64_t n, int64_t* __restrict__ sorted_rows,
                                    int64_t* __restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = (int64_t)pos[i];
    sorted_rows[i] = __ldg(rows + p);
    perm[i] = p;
  }
}

template <typename T>
__global__ void scatter_kernel(const T* __restrict__ in, const int64_t* __restrict__ perm,
                               int64_t n, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[__ldg(perm + i)] = in[i];
}

template <typename K>
static int sort_pairs(const int64_t* rows, int64_t n, int bits, int shift, int64_t* sorted_rows,
                      int64_t* perm, cudaStream_t s) {
  K* buf = nullptr;
  BSB_CUDA(cudaMallocAsync(&buf, (size_t)n * sizeof(K) * 4, s));
  K *k_in = buf, *k_out = buf + n, *v_in = buf + 2 * n, *v_out = buf + 3 * n;
  make_pairs_kernel<K><<<gather_grid(n, 256), 256, 0, s>>>(rows, n, shift, k_in, v_in);
  BSB_LAUNCH_CHECK();
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, v_in, v_out, n, 0, bits, s);
  void* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, tb + 16, s));
  cub::DeviceRadixSort::SortPairs(tmp, tb, k_in, k_out, v_in, v_out, n, 0, bits, s);
  BSB_LAUNCH_CHECK();
  unpack_pairs_kernel<K><<<gather_grid(n, 256), 256, 0, s>>>(rows, v_out, n, sorted_rows, perm);
  BSB_LAUNCH_CHECK();
  BSB_CUDA(cudaFreeAsync(tmp, s));
  BSB_CUDA(cudaFreeAsync(buf, s));
  return BSB_OK;
}


// --- bucket-ordered (row, position) pairs ------------------------------------
// The fast form of the above for lists of < 2^32 ids over columns of < 2^32
// rows: the gather needs locality, not order, so the ids are only PARTITIONED
// by row bucket (2^kPairBucketBits buckets of consecutive rows at most) into
// 8-byte pairs row | position << 32, and the lookup kernels read the pairs and
// write their output at `position` themselves (no sorted id array, no perm
// array, no scatter pass).  Three kernels: a histogram over the buckets, then
// two partition passes (the bucket's top kPairTopBits, then all of its bits
// inside each top group) -- each pass stages a chunk of kPairChunk pairs in
// shared memory ordered by bin and reserves the bin's global range with one
// atomicAdd per (chunk, bin), so global writes are runs of ~chunk / bins
// pairs.  The order of pairs inside a bucket depends on the atomics; the
// looked-up output does not (every pair carries its position).
constexpr int kPairBucketBits = 13;
constexpr int kPairTopBits = 7;
constexpr int kPairMaxBins = 1 << kPairTopBits;  // bins of one pass
constexpr int kPairChunk = 4096;
constexpr int kPairThreads = 512;
constexpr int kPairPer = kPairChunk / kPairThreads;
constexpr uint32_t kPairBadRow = 0xffffffffu;  // an id outside [0, n_rows): never a row

static int g_pair_bits = kPairBucketBits;  // bsb_tune("pair_bits"): bucket bits (1..13)
void set_pair_bits(int64_t v) {
  g_pair_bits = v < 1 || v > kPairBucketBits ? kPairBucketBits : (int)v;
}

struct PairPlan {
  int shift;      // bucket = min(row >> shift, n_buckets - 1)
  int n_buckets;  // 2^bits
  int sub_bits;   // bits of the second pass (0: one pass)
};

__device__ __forceinline__ uint32_t pair_bucket(uint32_t row, const PairPlan& pl) {
  const uint32_t b = row >> pl.shift;
  return b < (uint32_t)pl.n_buckets ? b : (uint32_t)pl.n_buckets - 1;
}

__device__ __forceinline__ uint32_t pair_row(int64_t r, int64_t n_rows) {
  return (uint64_t)r < (uint64_t)n_rows ? (uint32_t)r : kPairBadRow;
}

__global__ void __launch_bounds__(1024)
pair_hist_kernel(const int64_t* __restrict__ rows, int64_t n, int64_t n_rows, PairPlan pl,
                 uint32_t* __restrict__ hist, const uint32_t* __restrict__ gate) {
  __shared__ uint32_t h[1 << kPairBucketBits];
  if (gate_closed(gate, true)) return;
  for (int b = threadIdx.x; b < pl.n_buckets; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthr)
    atomicAdd(&h[pair_bucket(pair_row(__ldg(rows + i), n_rows), pl)], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < pl.n_buckets; b += blockDim.x)
    if (h[b]) atomicAdd(hist + b, h[b]);
}

// hist[n_buckets] -> cur2[b] = exclusive prefix (the bucket's first pair),
// cur1[g] / seg[g] = the first pair of top group g, seg[n_groups] = n.
__global__ void __launch_bounds__(1024)
pair_offsets_kernel(const uint32_t* __restrict__ hist, PairPlan pl, uint32_t n,
                    uint32_t* __restrict__ cur1, uint32_t* __restrict__ cur2,
                    uint32_t* __restrict__ seg, uint32_t* __restrict__ seg1,
                    const uint32_t* __restrict__ gate) {
  __shared__ uint32_t wsum[32];
  if (gate_closed(gate, true)) return;
  constexpr int kPer = (1 << kPairBucketBits) / 1024;
  uint32_t c[kPer], tot = 0;
  const int b0 = threadIdx.x * kPer;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    c[k] = b0 + k < pl.n_buckets ? hist[b0 + k] : 0u;
    tot += c[k];
  }
  uint32_t inc = tot;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, inc, d);
    if ((threadIdx.x & 31) >= d) inc += v;
  }
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = inc;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t w = wsum[threadIdx.x], wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, wi, d);
      if (threadIdx.x >= d) wi += v;
    }
    wsum[threadIdx.x] = wi - w;
  }
  __syncthreads();
  uint32_t ex = wsum[threadIdx.x >> 5] + inc - tot;
  const int gmask = (1 << pl.sub_bits) - 1;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int b = b0 + k;
    if (b < pl.n_buckets) {
      cur2[b] = ex;
      if ((b & gmask) == 0) {
        cur1[b >> pl.sub_bits] = ex;
        seg[b >> pl.sub_bits] = ex;
      }
    }
    ex += c[k];
  }
  if (threadIdx.x == 0) {
    seg[pl.n_buckets >> pl.sub_bits] = n;
    seg1[0] = 0;  // the first pass's single segment: the whole list
    seg1[1] = n;
  }
}

// One partition pass.  FIRST: src = the caller's int64 ids (one segment, the
// whole list), bin = bucket >> sub_bits, cursors cur1; else src = the first
// pass's pairs, segment g = top group g, bin = bucket (cursors cur2).  A chunk
// is contiguous in src: one elected thread fetches the NEXT chunk with a 1-D
// TMA bulk copy into the stage buffer while this chunk is ranked, placed and
// written (the kernel was bound by the chunk's load latency before: half of
// its stall samples sat on the first use of the loaded ids).
constexpr int kPairSmemBytes = (2 * kPairChunk + 2) * 8;

template <bool FIRST>
__global__ void __launch_bounds__(kPairThreads, 3)
pair_pass_kernel(const void* __restrict__ src, uint64_t* __restrict__ dst, int64_t n_rows,
                 PairPlan pl, const uint32_t* __restrict__ seg, int n_seg,
                 uint32_t* __restrict__ cursor, const uint32_t* __restrict__ gate) {
  extern __shared__ __align__(16) uint64_t pair_smem[];
  if (gate_closed(gate, true)) return;
  uint64_t* stage = pair_smem;                      // kPairChunk + 2: the TMA destination
  uint64_t* pair_buf = pair_smem + kPairChunk + 2;  // kPairChunk pairs ordered by bin
  __shared__ uint64_t bar;
  __shared__ uint32_t cnt[kPairMaxBins], lofs[kPairMaxBins], delta[kPairMaxBins];
  __shared__ uint32_t item0[kPairMaxBins + 1];  // first work item of every segment
  __shared__ uint32_t wtot[kPairMaxBins / 32];
  const int tid = threadIdx.x;
  const int nbins = FIRST ? (pl.n_buckets >> pl.sub_bits) : (1 << pl.sub_bits);
  if (tid == 0) {
    uint32_t acc = 0;
    for (int g = 0; g < n_seg; ++g) {
      item0[g] = acc;
      acc += (seg[g + 1] - seg[g] + kPairChunk - 1) / kPairChunk;
    }
    item0[n_seg] = acc;
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t n_items = item0[n_seg];
  const uint64_t* src64 = static_cast<const uint64_t*>(src);

  // work item -> segment, first element, length
  auto locate = [&](uint32_t item, int& g, uint32_t& base, uint32_t& len) {
    int lo = 0, hi = n_seg;  // last segment with item0 <= item
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (item0[mid] <= item) lo = mid; else hi = mid;
    }
    g = lo;
    base = seg[g] + (item - item0[g]) * kPairChunk;
    len = min((uint32_t)kPairChunk, seg[g + 1] - base);
  };
  // Start the bulk copy of a chunk (16-byte aligned source and size: the
  // copy starts one element early when the chunk does not; the first pass's
  // buffer is the caller's, so there only exactly aligned chunks are copied).
  auto fetch = [&](uint32_t base, uint32_t len, uint32_t& mis) -> bool {
    const uint64_t* p = src64 + base;
    mis = (uint32_t)((reinterpret_cast<uintptr_t>(p) >> 3) & 1);
    const bool bulk = FIRST ? (mis == 0 && (len & 1) == 0) : true;
    if (bulk && tid == 0) {
      const uint32_t bytes = ((len + mis + 1) & ~1u) * 8;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bar, bytes);
      bulk_g2s(stage, p - mis, bytes, &bar);
    }
    return bulk;
  };

  uint32_t item = blockIdx.x, parity = 0;
  int g = 0;
  uint32_t base = 0, len = 0, mis = 0;
  bool bulk = false;
  if (item < n_items) {
    locate(item, g, base, len);
    bulk = fetch(base, len, mis);
  }
  while (item < n_items) {
    if (tid < kPairMaxBins) cnt[tid] = 0;
    if (bulk) {
      mbar_wait(&bar, parity);
      parity ^= 1;
    }
    uint64_t pr[kPairPer];
#pragma unroll
    for (int k = 0; k < kPairPer; ++k) {
      const uint32_t i = k * kPairThreads + tid;
      if (i < len) pr[k] = bulk ? stage[mis + i] : __ldg(src64 + base + i);
    }
    __syncthreads();  // the stage is read, cnt is zero
    const int g_cur = g;
    const uint32_t base_cur = base, len_cur = len;
    item += gridDim.x;
    if (item < n_items) {
      locate(item, g, base, len);
      bulk = fetch(base, len, mis);
    }
    uint32_t rank[kPairPer];
#pragma unroll
    for (int k = 0; k < kPairPer; ++k) {
      const uint32_t i = k * kPairThreads + tid;
      if (i < len_cur) {
        if (FIRST)
          pr[k] = (uint64_t)pair_row((int64_t)pr[k], n_rows) | ((uint64_t)(base_cur + i) << 32);
        const uint32_t b = pair_bucket((uint32_t)pr[k], pl);
        const uint32_t bin = FIRST ? (b >> pl.sub_bits) : (b & ((1u << pl.sub_bits) - 1));
        rank[k] = atomicAdd(&cnt[bin], 1u) | (bin << 16);
      }
    }
    __syncthreads();
    if (tid < kPairMaxBins) {  // exclusive scan of the bin counts, global reservation
      const uint32_t c = tid < nbins ? cnt[tid] : 0u;
      uint32_t inc = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, inc, d);
        if ((tid & 31) >= d) inc += v;
      }
      if ((tid & 31) == 31) wtot[tid >> 5] = inc;
      // the 4 warps of this branch meet at a named barrier (the other warps go on)
      asm volatile("bar.sync 1, %0;" ::"n"(kPairMaxBins));
      uint32_t ex = inc - c;
#pragma unroll
      for (int w = 0; w < kPairMaxBins / 32; ++w)
        if (w < (tid >> 5)) ex += wtot[w];
      lofs[tid] = ex;
      uint32_t gb = 0;
      if (c) gb = atomicAdd(cursor + (FIRST ? tid : (g_cur << pl.sub_bits) + tid), c);
      delta[tid] = gb - ex;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPairPer; ++k) {
      const uint32_t i = k * kPairThreads + tid;
      if (i < len_cur) pair_buf[lofs[rank[k] >> 16] + (rank[k] & 0xffffu)] = pr[k];
    }
    __syncthreads();
    for (uint32_t i = tid; i < len_cur; i += kPairThreads) {
      const uint64_t p = pair_buf[i];
      const uint32_t b = pair_bucket((uint32_t)p, pl);
      const uint32_t bin = FIRST ? (b >> pl.sub_bits) : (b & ((1u << pl.sub_bits) - 1));
      dst[delta[bin] + i] = p;
    }
    // the next iteration's first barrier orders these reads of pair_buf /
    // delta before their next writes
  }
}

}  // namespace bsb

using namespace bsb;

extern "C" int bsb_rows_sort(const int64_t* rows, int64_t n_ids, int64_t n_rows,
                             int64_t* sorted_rows, int64_t* perm, int32_t* was_sorted,
                             void* stream) {
  if (!rows || !sorted_rows || !perm || !was_sorted || n_ids < 0 || n_rows <= 0)
    return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  *was_sorted = 1;
  if (n_ids < 2) return BSB_OK;
  unsigned int* bad = nullptr;
  BSB_CUDA(cudaMallocAsync(&bad, 4, s));
  BSB_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  // A sampled order check (adjacent pairs at 4096 spread positions): a
  // wrongly "sorted" verdict only skips an optimisation, never changes
  // results, and the check stays a few microseconds for any list length.
  rows_sample_check_kernel<<<4, 1024, 0, s>>>(rows, n_ids, bad);
  BSB_LAUNCH_CHECK();
  unsigned int h = 0;
  BSB_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(bad, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (!h) return BSB_OK;
  *was_sorted = 0;
  int bits = 1;
  while (bits < 64 && ((uint64_t)(n_rows - 1) >> bits) != 0) ++bits;
  // Order by 2^shift-row bucket, at most 2^16 buckets (two radix passes):
  // a bucket's ids touch one contiguous region of every array, which is all
  // the locality the gather needs (ids inside a bucket keep input order).
  const int shift = bits > kBucketBits ? bits - kBucketBits : 0;
  if (n_ids <= (int64_t)UINT32_MAX)
    return sort_pairs<uint32_t>(rows, n_ids, bits - shift, shift, sorted_rows, perm, s);
  return sort_pairs<unsigned long long>(rows, n_ids, bits - shift, shift, sorted_rows, perm, s);
}

namespace bsb {

// One CTA: 4096 sampled adjacent pairs, verdict + 1 into a host-mapped word.
__global__ void __launch_bounds__(1024)
rows_sample_poll_kernel(const int64_t* __restrict__ rows, int64_t n,
                        volatile uint32_t* __restrict__ flag) {
  bool b = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = (n - 1) * (int64_t)(threadIdx.x + 1024 * q) / 4096;
    b |= i + 1 < n && __ldg(rows + i + 1) < __ldg(rows + i);
  }
  const int any = __syncthreads_or(b);
  if (threadIdx.x == 0) {
    *flag = any ? 2u : 1u;
    __threadfence_system();
  }
}

int rows_order_poll(const int64_t* rows, int64_t n_ids, cudaStream_t s) {
  constexpr int kSlots = 1024;
  struct Ring {
    volatile uint32_t* host = nullptr;
    uint32_t* dev = nullptr;
    Ring() {
      void* h = nullptr;
      if (cudaHostAlloc(&h, kSlots * sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess) return;
      void* d = nullptr;
      if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return;
      host = static_cast<volatile uint32_t*>(h);
      dev = static_cast<uint32_t*>(d);
    }
  };
  static Ring ring;
  static std::atomic<uint32_t> next{0};
  if (!ring.dev || n_ids < 2) return -1;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return -1;
  // only on an idle stream: behind queued work the poll would wait for all of it
  if (cudaStreamQuery(s) != cudaSuccess) {
    cudaGetLastError();  // cudaErrorNotReady is not an error
    return -1;
  }
  const uint32_t slot = next.fetch_add(1) % kSlots;
  ring.host[slot] = 0u;
  rows_sample_poll_kernel<<<1, 1024, 0, s>>>(rows, n_ids, ring.dev + slot);
  if (cudaGetLastError() != cudaSuccess) return -1;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const uint32_t v = ring.host[slot];
    if (v) return (int)v - 1;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(500)) return -1;
  }
}

void rows_order_check_launch(const int64_t* rows, int64_t n_ids, uint32_t* unsorted_dev,
                             cudaStream_t s) {
  rows_sample_check_kernel<<<4, 1024, 0, s>>>(rows, n_ids, unsorted_dev);
}

int rows_order_check(const int64_t* rows, int64_t n_ids, uint32_t* unsorted_dev, cudaStream_t s) {
  BSB_CUDA(cudaMemsetAsync(unsorted_dev, 0, 4, s));
  if (n_ids >= 2) {
    rows_sample_check_kernel<<<4, 1024, 0, s>>>(rows, n_ids, unsorted_dev);
    BSB_LAUNCH_CHECK();
  }
  return BSB_OK;
}

int rows_bucket_gated(const int64_t* rows, int64_t n_ids, int64_t n_rows, uint64_t* pairs,
                      const uint32_t* gate, cudaStream_t s) {
  int bits = 1;
  while (bits < 32 && ((uint64_t)(n_rows - 1) >> bits) != 0) ++bits;
  PairPlan pl;
  // buckets of at least 2^10 rows: finer ones add nothing to sector sharing
  int bbits = bits - 10;
  if (bbits > g_pair_bits) bbits = g_pair_bits;
  if (bbits < 1) bbits = 1;
  pl.shift = bits - bbits;
  pl.n_buckets = 1 << bbits;
  pl.sub_bits = bbits > kPairTopBits ? bbits - kPairTopBits : 0;
  const int n_groups = pl.n_buckets >> pl.sub_bits;
  // scratch: hist | cur1 | cur2 | seg | first-pass pairs
  const size_t words = (size_t)pl.n_buckets * 2 + 2 * kPairMaxBins + 8;
  const size_t head = (words * 4 + 255) & ~(size_t)255;
  uint8_t* scratch = nullptr;
  BSB_CUDA(cudaMallocAsync(&scratch, head + (pl.sub_bits ? (size_t)n_ids * 8 + 16 : 0), s));
  uint32_t* hist = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* cur2 = hist + pl.n_buckets;
  uint32_t* cur1 = cur2 + pl.n_buckets;
  uint32_t* seg = cur1 + kPairMaxBins;
  uint64_t* mid = reinterpret_cast<uint64_t*>(scratch + head);
  BSB_CUDA(cudaMemsetAsync(hist, 0, (size_t)pl.n_buckets * 4, s));
  static bool attr_done = false;
  if (!attr_done) {
    BSB_CUDA(cudaFuncSetAttribute(pair_pass_kernel<true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmemBytes));
    BSB_CUDA(cudaFuncSetAttribute(pair_pass_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmemBytes));
    attr_done = true;
  }
  const int64_t chunks = (n_ids + kPairChunk - 1) / kPairChunk;
  int gh = (int)((n_ids + 1024 * 8 - 1) / (1024 * 8));
  if (gh > sm_count() * 2) gh = sm_count() * 2;
  if (gh < 1) gh = 1;
  pair_hist_kernel<<<gh, 1024, 0, s>>>(rows, n_ids, n_rows, pl, hist, gate);
  BSB_LAUNCH_CHECK();
  uint32_t* seg1 = seg + kPairMaxBins + 2;  // the first pass's one segment {0, n}
  pair_offsets_kernel<<<1, 1024, 0, s>>>(hist, pl, (uint32_t)n_ids, cur1, cur2, seg, seg1,
                                         gate);
  BSB_LAUNCH_CHECK();
  int gp = (int)(chunks < (int64_t)sm_count() * 3 ? chunks : (int64_t)sm_count() * 3);
  pair_pass_kernel<true><<<gp, kPairThreads, kPairSmemBytes, s>>>(
      rows, pl.sub_bits ? mid : pairs, n_rows, pl, seg1, 1, cur1, gate);
  BSB_LAUNCH_CHECK();
  if (pl.sub_bits) {
    int gp2 = (int)(chunks + n_groups < (int64_t)sm_count() * 3 ? chunks + n_groups
                                                                 : (int64_t)sm_count() * 3);
    pair_pass_kernel<false><<<gp2, kPairThreads, kPairSmemBytes, s>>>(
        mid, pairs, n_rows, pl, seg, n_groups, cur2, gate);
    BSB_LAUNCH_CHECK();
  }
  BSB_CUDA(cudaFreeAsync(scratch, s));
  return BSB_OK;
}

}  // namespace bsb

extern "C" int bsb_rows_bucket(const int64_t* rows, int64_t n_ids, int64_t n_rows,
                               uint64_t* pairs, uint32_t* unsorted_dev, void* stream) {
  if (!rows || !pairs || n_ids < 0 || n_rows <= 0) return BSB_EINVAL;
  if (n_ids >= (int64_t)UINT32_MAX || n_rows >= (int64_t)UINT32_MAX) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  if (unsorted_dev) {
    // the sampled order check of bsb_rows_sort, its verdict left on the
    // device: every kernel below exits at once when the list looks ascending
    const int rc = rows_order_check(rows, n_ids, unsorted_dev, s);
    if (rc) return rc;
  }
  if (n_ids == 0) return BSB_OK;
  return rows_bucket_gated(rows, n_ids, n_rows, pairs, unsorted_dev, s);
}

extern "C" int bsb_scatter(const void* in, const int64_t* perm, int64_t n, int32_t elem_bytes,
                           void* out, void* stream) {
  if ((n > 0 && (!in || !perm || !out)) || n < 0) return BSB_EINVAL;
  if (n == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  const int g = gather_grid(n, 256);
  if (elem_bytes == 4)
    scatter_kernel<uint32_t><<<g, 256, 0, s>>>(static_cast<const uint32_t*>(in), perm, n,
                                               static_cast<uint32_t*>(out));
  else if (elem_bytes == 8)
    scatter_kernel<unsigned long long><<<g, 256, 0, s>>>(
        static_cast<const unsigned long long*>(in), perm, n,
        static_cast<unsigned long long*>(out));
  else
    return BSB_EINVAL;
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}
