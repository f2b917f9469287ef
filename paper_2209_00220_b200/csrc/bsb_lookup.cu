// bsb_lookup.cu -- row lookups (ByteSlice / PP-VBS), decode, bitvector
// compaction and word-level bitvector algebra.
#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "bsb_common.cuh"

namespace bsb {

static int grid_for_l(int64_t items, int threads, int cap = 148 * 16) {
  int64_t g = (items + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// lookup_byteslice (byteslice.py:143-158) + decode_ranks (dictionary.py:413-414).
// Each thread takes kIdsPerThread ids per iteration so their random sector
// loads are in flight together.
constexpr int kIdsPerThread = 4;
// PP-VBS row ids: a row gathers up to K sectors of 8 registers each
constexpr int kVbsIds = 1;
// ByteSlice row ids: one id per thread at a time with all K sector loads in
// flight together (8 registers each) keeps more threads resident
constexpr int kBsIds = 1;

// PAIRS: ids = bucket-ordered row | position << 32 pairs (bsb_rows_bucket);
// the kernels write pair i's result at i and pair_scatter_kernel moves it to
// its position.
template <bool PAIRS>
__device__ __forceinline__ int64_t id_at(const void* __restrict__ ids, int64_t i) {
  if (PAIRS)  // 0xffffffff (an id out of range) stays out of range
    return (int64_t)(uint32_t)__ldg(static_cast<const unsigned long long*>(ids) + i);
  return __ldg(static_cast<const long long*>(ids) + i);
}

__device__ __forceinline__ void emit(uint64_t* oc, int64_t* ov, int32_t* ov32, int64_t pos,
                                     uint64_t code_out, int64_t v) {
  if (oc) oc[pos] = code_out;
  if (ov) ov[pos] = v;
  if (ov32) ov32[pos] = (int32_t)v;
}

// out[position of pair i] = in[i]: the results of a pair lookup (pair order)
// back to the caller's order.  A kernel of its own: the same stores issued
// from inside the gather measured 2.5x slower (B200: 2^24 int32 results, 409
// MB written and 330 MB more read than the 64 MB the output has -- the column
// sectors streaming through L2 evict the partially written output sectors),
// L2 evict_last / evict_first policies on the stores and the streamed loads
// changed nothing in either form.
template <typename T>
__global__ void pair_scatter_kernel(const unsigned long long* __restrict__ pairs,
                                    const T* __restrict__ in, int64_t n, T* __restrict__ out,
                                    const uint32_t* __restrict__ gate) {
  if (gate_closed(gate, true)) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[__ldg(pairs + i) >> 32] = in[i];
}

// Temporaries of a pair lookup: one per requested output, in pair order.
struct PairOut {
  uint64_t* oc = nullptr;
  int64_t* ov = nullptr;
  int32_t* ov32 = nullptr;
};
static int pair_out_alloc(PairOut& t, int64_t n, bool oc, bool ov, bool ov32, cudaStream_t s) {
  if (oc) BSB_CUDA(cudaMallocAsync(&t.oc, (size_t)n * 8, s));
  if (ov) BSB_CUDA(cudaMallocAsync(&t.ov, (size_t)n * 8, s));
  if (ov32) BSB_CUDA(cudaMallocAsync(&t.ov32, (size_t)n * 4, s));
  return BSB_OK;
}
static int pair_out_scatter(PairOut& t, const uint64_t* pairs, int64_t n, uint64_t* oc,
                            int64_t* ov, int32_t* ov32, const uint32_t* gate, cudaStream_t s) {
  const int g = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
  const unsigned long long* pp = reinterpret_cast<const unsigned long long*>(pairs);
  if (t.oc) pair_scatter_kernel<uint64_t><<<g, 256, 0, s>>>(pp, t.oc, n, oc, gate);
  if (t.ov) pair_scatter_kernel<int64_t><<<g, 256, 0, s>>>(pp, t.ov, n, ov, gate);
  if (t.ov32) pair_scatter_kernel<int32_t><<<g, 256, 0, s>>>(pp, t.ov32, n, ov32, gate);
  BSB_LAUNCH_CHECK();
  if (t.oc) BSB_CUDA(cudaFreeAsync(t.oc, s));
  if (t.ov) BSB_CUDA(cudaFreeAsync(t.ov, s));
  if (t.ov32) BSB_CUDA(cudaFreeAsync(t.ov32, s));
  return BSB_OK;
}

// 8 CTAs of 256 threads per SM (<= 32 registers): the gather lives on its
// loads in flight; at 34 registers (6 CTAs) the sorted-id gather ran 212 us
// instead of 173 us.
template <bool PAIRS>
__global__ void __launch_bounds__(256, 8) bs_lookup_kernel(const uint8_t* __restrict__ slices, int64_t stride, int K,
                                 int width, const void* __restrict__ rows, int64_t n_ids,
                                 uint64_t* __restrict__ out_codes,
                                 const int64_t* __restrict__ rank_values,
                                 int64_t* __restrict__ out_values,
                                 int32_t* __restrict__ out_values32, int64_t n_rows,
                                 unsigned int* __restrict__ err,
                                 const uint32_t* __restrict__ gate, bool want) {
  if (gate_closed(gate, want)) return;
  const int shift = 8 * K - width;
  bool oob = false;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n_ids;
       i0 += nthr * kBsIds) {
    int64_t blk[kBsIds];
    int lr[kBsIds];
    uint64_t c[kBsIds];
#pragma unroll
    for (int u = 0; u < kBsIds; ++u) {
      const int64_t i = i0 + u * nthr;
      int64_t r = i < n_ids ? id_at<PAIRS>(rows, i) : 0;
      if ((uint64_t)r >= (uint64_t)n_rows) {  // IndexError in the reference; never read it
        oob = true;
        r = 0;
      }
      blk[u] = r >> 5;
      lr[u] = (int)(r & 31);
      c[u] = 0;
    }
#pragma unroll
    for (int j = 0; j < kMaxLevels; ++j) {
      if (j >= K) break;
      uint32_t w[kBsIds][8];
#pragma unroll
      for (int u = 0; u < kBsIds; ++u) {
        if (i0 + u * nthr < n_ids) {
          ldg256_free(slices + (int64_t)j * stride + blk[u] * 32, w[u]);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) w[u][q] = 0;
        }
      }
#pragma unroll
      for (int u = 0; u < kBsIds; ++u) c[u] = (c[u] << 8) | bp_byte(w[u], lr[u]);
    }
#pragma unroll
    for (int u = 0; u < kBsIds; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i >= n_ids) break;
      const uint64_t cd = c[u] >> shift;
      // out_values32 without rank_values: codes that are the values (identity dictionary)
      const int64_t v = rank_values ? __ldg(rank_values + cd) : (int64_t)cd;
      emit(out_codes, rank_values ? out_values : nullptr, out_values32, i, cd, v);
    }
  }
  if (__any_sync(kFull, oob) && (threadIdx.x & 31) == 0) atomicOr(err, kErrIndex);
}

struct VbsLookupDesc {
  const uint8_t* bs1;
  const uint8_t* deep[kMaxLevels];
  const uint32_t* exist[kMaxLevels];
  const int64_t* dir[kMaxLevels];
  int64_t n_rows;
  int K;
  int mode;
};

static void fill_lookup_desc(VbsLookupDesc& d, const bsb_vbs* col) {
  std::memset(&d, 0, sizeof(d));
  d.bs1 = col->bs1;
  d.K = col->max_len;
  d.mode = col->deep_mode;
  d.n_rows = col->n_rows;
  for (int j = 0; j < kMaxLevels; ++j) {
    d.deep[j] = col->deep[j];
    d.exist[j] = col->exist[j];
    d.dir[j] = col->block_dir[j];
  }
}

// lookup_vbs (vbs.py:331-371) + decode_padded (dictionary.py:403-411)
__global__ void vbs_lookup_kernel(const __grid_constant__ VbsLookupDesc d,
                                  const int64_t* __restrict__ rows, int64_t n_ids,
                                  uint64_t* __restrict__ out_padded,
                                  const uint64_t* __restrict__ sorted_padded,
                                  const int64_t* __restrict__ dict_values, int64_t n_dict,
                                  int64_t* __restrict__ out_values,
                                  int32_t* __restrict__ out_values32,
                                  unsigned int* __restrict__ err,
                                  unsigned long long* __restrict__ level_counts) {
  const int K = d.K;
  unsigned long long lc[kMaxLevels];
#pragma unroll
  for (int j = 0; j < kMaxLevels; ++j) lc[j] = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ids;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = __ldg(rows + i);
    if ((uint64_t)r >= (uint64_t)d.n_rows) {  // IndexError in the reference; never read it
      atomicOr(err, kErrIndex);
      r = 0;
    }
    const int64_t b = r >> 5;
    const int lr = (int)(r & 31);
    uint64_t code = (uint64_t)bp_row_byte(d.bs1 + b * 32, lr) << (8 * (K - 1));
    const uint32_t below = (1u << lr) - 1u;
    lc[0] += 1;
    int64_t pos2 = 0;
    if (d.mode != BSB_DEEP_PACKED && K >= 2) {
      const uint32_t w2 = __ldg(d.exist[1] + b);
      if ((w2 >> lr) & 1u) pos2 = __ldg(d.dir[1] + b) + __popc(w2 & below);
    }
    for (int j = 2; j <= K; ++j) {
      const uint32_t w = __ldg(d.exist[j - 1] + b);
      if (!((w >> lr) & 1u)) break;  // lengths are nested: no deeper byte
#pragma unroll
      for (int q = 1; q < kMaxLevels; ++q)
        if (q == j - 1) lc[q] += 1;
      uint64_t byte;
      if (d.mode == BSB_DEEP_SLICED) {
        byte = bp_row_byte(d.deep[j - 1] + (pos2 >> 5) * 32, (int)(pos2 & 31));
      } else {
        const int64_t pos = __ldg(d.dir[j - 1] + b) + __popc(w & below);
        byte = __ldg(d.deep[j - 1] + pos);
      }
      code |= byte << (8 * (K - j));
    }
    if (out_padded) out_padded[i] = code;
    if (sorted_padded) {
      // lower_bound over the strictly increasing padded codes
      int64_t lo = 0, hi = n_dict;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(sorted_padded + mid) < code)
          lo = mid + 1;
        else
          hi = mid;
      }
      int64_t v = 0;
      if (lo >= n_dict || __ldg(sorted_padded + lo) != code) {
        atomicOr(err, kErrNotFound);
      } else {
        v = __ldg(dict_values + lo);
      }
      if (out_values) out_values[i] = v;
      if (out_values32) out_values32[i] = (int32_t)v;
    }
  }
  if (level_counts) {
#pragma unroll
    for (int j = 0; j < kMaxLevels; ++j) {
      unsigned long long v = lc[j];
#pragma unroll
      for (int dd = 16; dd > 0; dd >>= 1) v += __shfl_xor_sync(kFull, v, dd);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(level_counts + j, v);
    }
  }
}

// --- bitvector -> ascending row ids (bitvector.py:71-72) ---------------------
// Both kernels take a SUPER-TILE of 4 tiles (128 words, 4096 rows) per warp
// iteration, lane l holding the 4 consecutive words 4l .. 4l+3 from one
// 16-byte load, two super-tiles' loads in flight per iteration: with one
// 4-byte load per lane and iteration (the first form) the 64 MB of a 2^29-row
// selection took 27 + 69 us -- ~0.8 TB/s, all load latency -- inside every
// cfg5 step.
__device__ __forceinline__ uint4 sel_words4(const uint32_t* __restrict__ words, int64_t w0,
                                            int64_t nb) {
  if (w0 + 4 <= nb) return __ldg(reinterpret_cast<const uint4*>(words + w0));
  uint4 v = make_uint4(0u, 0u, 0u, 0u);  // the column's last words
  if (w0 < nb) v.x = __ldg(words + w0);
  if (w0 + 1 < nb) v.y = __ldg(words + w0 + 1);
  if (w0 + 2 < nb) v.z = __ldg(words + w0 + 2);
  return v;
}

// tile_counts[t] = set bits of tile t.  words must be 16-byte aligned.
__global__ void tile_popc_kernel(const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
                                 int64_t* __restrict__ tile_counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsuper = (ntiles + 3) >> 2;
  for (int64_t s0 = warp * 2; s0 < nsuper; s0 += nwarps * 2) {
    uint4 v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) v[u] = sel_words4(words, (s0 + u) * 128 + lane * 4, nb);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      // a tile = 8 consecutive lanes (32 words): sum inside each group of 8
      unsigned c = __popc(v[u].x) + __popc(v[u].y) + __popc(v[u].z) + __popc(v[u].w);
      c += __shfl_xor_sync(kFull, c, 1);
      c += __shfl_xor_sync(kFull, c, 2);
      c += __shfl_xor_sync(kFull, c, 4);
      const int64_t t = (s0 + u) * 4 + (lane >> 3);
      if ((lane & 7) == 0 && t < ntiles) tile_counts[t] = c;
    }
  }
}

__global__ void __launch_bounds__(256, 8) tile_emit_kernel(const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
                                 const int64_t* __restrict__ tile_incl, int64_t row_offset,
                                 const int64_t* __restrict__ base_dev,
                                 int64_t* __restrict__ rows_out) {
  if (base_dev) rows_out += __ldg(base_dev);  // compaction into a shared id array
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsuper = (ntiles + 3) >> 2;
  for (int64_t s0 = warp * 2; s0 < nsuper; s0 += nwarps * 2) {
    uint4 v[2];
    int64_t before[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      v[u] = sel_words4(words, (s0 + u) * 128 + lane * 4, nb);
      const int64_t t0 = (s0 + u) * 4;  // selected rows before the super-tile
      before[u] = (t0 > 0 && t0 <= ntiles) ? __ldg(tile_incl + t0 - 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t wq[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
      const uint32_t c = __popc(wq[0]) + __popc(wq[1]) + __popc(wq[2]) + __popc(wq[3]);
      if (!__any_sync(kFull, c != 0)) continue;
      const uint32_t incl = warp_incl_scan(c);
      int64_t pos = before[u] + (incl - c);
      const int64_t b0 = (s0 + u) * 128 + lane * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t w = wq[q];
        while (w) {
          const int bit = __ffs(w) - 1;
          w &= w - 1;
          rows_out[pos++] = row_offset + (b0 + q) * 32 + bit;
        }
      }
    }
  }
}

// the first forms (any alignment of words): one word per lane and iteration
__global__ void tile_popc1_kernel(const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
                                  int64_t* __restrict__ tile_counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < ntiles; t += nwarps) {
    const int64_t b = t * 32 + lane;
    unsigned c = b < nb ? __popc(__ldg(words + b)) : 0u;
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) tile_counts[t] = c;
  }
}

__global__ void tile_emit1_kernel(const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
                                  const int64_t* __restrict__ tile_incl, int64_t row_offset,
                                  const int64_t* __restrict__ base_dev,
                                  int64_t* __restrict__ rows_out) {
  if (base_dev) rows_out += __ldg(base_dev);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = warp; t < ntiles; t += nwarps) {
    const int64_t b = t * 32 + lane;
    uint32_t w = b < nb ? __ldg(words + b) : 0u;
    const uint32_t c = __popc(w);
    const uint32_t incl = warp_incl_scan(c);
    const int64_t base = (t ? tile_incl[t - 1] : 0) + (incl - c);
    int64_t pos = base;
    while (w) {
      const int bit = __ffs(w) - 1;
      w &= w - 1;
      rows_out[pos++] = row_offset + b * 32 + bit;
    }
  }
}

// tile counts of a selection (either form, by the alignment of words)
static void launch_tile_popc(const uint32_t* words, int64_t nb, int64_t ntiles, int64_t* tc,
                             cudaStream_t s) {
  if ((reinterpret_cast<uintptr_t>(words) & 15u) == 0) {
    const int64_t nsuper = (ntiles + 3) / 4;
    tile_popc_kernel<<<grid_for_l((nsuper + 1) / 2 * 32, 256), 256, 0, s>>>(words, nb, ntiles, tc);
  } else {
    tile_popc1_kernel<<<grid_for_l(ntiles * 32, 256), 256, 0, s>>>(words, nb, ntiles, tc);
  }
}

__global__ void combine_kernel(int op, const uint32_t* __restrict__ a,
                               const uint32_t* __restrict__ b, uint32_t* __restrict__ out,
                               int64_t n_rows, int64_t nb) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = a[i];
    uint32_t v;
    switch (op) {
      case 0: v = x & b[i]; break;
      case 1: v = x | b[i]; break;
      case 2: v = ~x; break;
      default: v = x & ~b[i]; break;
    }
    out[i] = v & tail_valid(i, n_rows);
  }
}

__global__ void popcount_kernel(const uint32_t* __restrict__ w, int64_t nb,
                                unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x)
    c += __popc(w[i]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

static int bits_to_rows_impl(const uint32_t* words, int64_t n_rows, int64_t row_offset,
                             const int64_t* base_dev, int64_t* rows_out, uint64_t* n_out_dev, int64_t* n_out_host,
                             cudaStream_t s) {
  const int64_t nb = (n_rows + 31) / 32;
  const int64_t ntiles = (nb + 31) / 32;
  int64_t* tc = nullptr;
  BSB_CUDA(cudaMallocAsync(&tc, (ntiles * 2 + 2) * sizeof(int64_t), s));
  int64_t* incl = tc + ntiles + 1;
  launch_tile_popc(words, nb, ntiles, tc, s);
  BSB_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, tc, incl, ntiles, s);
  void* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, tc, incl, ntiles, s);
  BSB_LAUNCH_CHECK();
  if (rows_out) {
    if ((reinterpret_cast<uintptr_t>(words) & 15u) == 0) {
      const int64_t nsuper = (ntiles + 3) / 4;
      tile_emit_kernel<<<grid_for_l((nsuper + 1) / 2 * 32, 256), 256, 0, s>>>(
          words, nb, ntiles, incl, row_offset, base_dev, rows_out);
    } else {
      tile_emit1_kernel<<<grid_for_l(ntiles * 32, 256), 256, 0, s>>>(
          words, nb, ntiles, incl, row_offset, base_dev, rows_out);
    }
    BSB_LAUNCH_CHECK();
  }
  if (n_out_dev)
    BSB_CUDA(cudaMemcpyAsync(n_out_dev, incl + ntiles - 1, 8, cudaMemcpyDeviceToDevice, s));
  if (n_out_host)
    BSB_CUDA(cudaMemcpyAsync(n_out_host, incl + ntiles - 1, 8, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(tmp, s));
  BSB_CUDA(cudaFreeAsync(tc, s));
  if (n_out_host) BSB_CUDA(cudaStreamSynchronize(s));
  return BSB_OK;
}

}  // namespace bsb

using namespace bsb;

// Reads the device error word of a row-id lookup (synchronises) and maps it
// to a status: an out-of-range id wins over an absent code.
static int err_status(unsigned int h) {
  if (h & kErrIndex) {
    set_error_msg("row id out of range");
    return BSB_EINDEX;
  }
  if (h & kErrNotFound) {
    set_error_msg("padded code not in dictionary");
    return BSB_ENOTFOUND;
  }
  return BSB_OK;
}

static int read_err(unsigned int* err, cudaStream_t s) {
  unsigned int h = 0;
  BSB_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(err, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  return err_status(h);
}

static int alloc_err(unsigned int** err, cudaStream_t s) {
  BSB_CUDA(cudaMallocAsync(err, 4, s));
  BSB_CUDA(cudaMemsetAsync(*err, 0, 4, s));
  return BSB_OK;
}

// pairs NULL: the row-id list `rows` as given.  Else the bucket-ordered pairs;
// with unsorted_dev (bsb_rows_bucket's verdict) both forms are launched and
// the one the verdict rules out exits at once.
// Scratch of the *_auto lookups: the pairs and the order verdict.
struct AutoScratch {
  uint64_t* pairs = nullptr;
  uint32_t* unsorted = nullptr;
};
static bool auto_fits(int64_t n_ids, int64_t n_rows) {
  return n_ids >= 2 && n_ids < (int64_t)UINT32_MAX && n_rows < (int64_t)UINT32_MAX;
}
// One allocation, one memset: pairs | verdict | error word.  (Forking the
// pair path onto a side stream, so that an ascending list's exiting kernels
// run beside its gather, measured no faster: the cost is host launch time.)
static int auto_begin(AutoScratch& a, const int64_t* rows, int64_t n_ids, unsigned int** err,
                      cudaStream_t s, bool check = true) {
  BSB_CUDA(cudaMallocAsync(&a.pairs, (size_t)n_ids * 8 + 16, s));
  a.unsorted = reinterpret_cast<uint32_t*>(a.pairs + n_ids);
  if (!*err) {
    *err = a.unsorted + 1;
    BSB_CUDA(cudaMemsetAsync(a.unsorted, 0, 8, s));
  } else {
    BSB_CUDA(cudaMemsetAsync(a.unsorted, 0, 4, s));
  }
  if (check && n_ids >= 2) {
    rows_order_check_launch(rows, n_ids, a.unsorted, s);
    BSB_LAUNCH_CHECK();
  }
  return BSB_OK;
}
// err_dev NULL: the error word lives in the scratch; read it, then free
static int auto_end(AutoScratch& a, unsigned int* err, bool own_err, cudaStream_t s) {
  unsigned int h = 0;
  if (own_err) BSB_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(a.pairs, s));
  if (!own_err) return BSB_OK;
  BSB_CUDA(cudaStreamSynchronize(s));
  return err_status(h);
}

static int bs_lookup_rows_impl(const bsb_byteslice* col, const int64_t* rows,
                               const uint64_t* pairs, const uint32_t* unsorted_dev,
                               int64_t n_ids, uint64_t* out_codes, const int64_t* rank_values,
                               int64_t* out_values, int32_t* out_values32, uint32_t* err_dev,
                               void* stream, bool automatic = false) {
  if (!col || n_ids < 0 || (n_ids > 0 && !rows && !pairs)) return BSB_EINVAL;
  if (pairs && unsorted_dev && !rows) return BSB_EINVAL;
  if (n_ids == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  const cudaStream_t ps = s;
  unsigned int* err = err_dev;
  AutoScratch au;
  automatic = automatic && auto_fits(n_ids, col->n_rows);
  // On an idle stream the host reads the order verdict itself (a poll of a
  // few microseconds) and launches only the form that applies; otherwise the
  // verdict stays on the device and both forms are launched, gated.
  const int polled = automatic ? rows_order_poll(rows, n_ids, s) : -1;
  if (polled == 0) automatic = false;  // ascending: the list as given
  if (automatic) {
    const int rc = auto_begin(au, rows, n_ids, &err, s, polled < 0);
    if (rc) return rc;
    pairs = au.pairs;
    unsorted_dev = polled < 0 ? au.unsorted : nullptr;
  } else if (!err) {
    const int rc = alloc_err(&err, s);
    if (rc) return rc;
  }
  const int g = grid_for_l((n_ids + kBsIds - 1) / kBsIds, 256);
  if (!pairs || unsorted_dev) {
    bs_lookup_kernel<false><<<g, 256, 0, s>>>(col->slices, col->stride, col->n_slices,
                                              col->width_bits, rows, n_ids, out_codes,
                                              rank_values, out_values, out_values32,
                                              col->n_rows, err, pairs ? unsorted_dev : nullptr,
                                              false);
    BSB_LAUNCH_CHECK();
  }
  if (automatic) {
    const int rc = rows_bucket_gated(rows, n_ids, col->n_rows, au.pairs, unsorted_dev, ps);
    if (rc) return rc;
  }
  if (pairs) {
    PairOut t;
    int rc = pair_out_alloc(t, n_ids, out_codes, rank_values && out_values, out_values32, ps);
    if (rc) return rc;
    bs_lookup_kernel<true><<<g, 256, 0, ps>>>(col->slices, col->stride, col->n_slices,
                                              col->width_bits, pairs, n_ids, t.oc, rank_values,
                                              t.ov, t.ov32, col->n_rows, err, unsorted_dev, true);
    BSB_LAUNCH_CHECK();
    rc = pair_out_scatter(t, pairs, n_ids, out_codes, out_values, out_values32, unsorted_dev,
                          ps);
    if (rc) return rc;
  }
  if (automatic) return auto_end(au, err, !err_dev, s);
  return err_dev ? BSB_OK : read_err(err, s);
}

extern "C" int bsb_byteslice_lookup_rows_auto(const bsb_byteslice* col, const int64_t* rows,
                                              int64_t n_ids, uint64_t* out_codes,
                                              const int64_t* rank_values, int64_t* out_values,
                                              int32_t* out_values32, uint32_t* err_dev,
                                              void* stream) {
  if (!rows && n_ids > 0) return BSB_EINVAL;
  return bs_lookup_rows_impl(col, rows, nullptr, nullptr, n_ids, out_codes, rank_values,
                             out_values, out_values32, err_dev, stream, true);
}

extern "C" int bsb_byteslice_lookup_rows(const bsb_byteslice* col, const int64_t* rows,
                                         int64_t n_ids, uint64_t* out_codes,
                                         const int64_t* rank_values, int64_t* out_values,
                                         int32_t* out_values32, uint32_t* err_dev,
                                         void* stream) {
  return bs_lookup_rows_impl(col, rows, nullptr, nullptr, n_ids, out_codes, rank_values,
                             out_values, out_values32, err_dev, stream);
}

extern "C" int bsb_byteslice_lookup_pairs(const bsb_byteslice* col, const uint64_t* pairs,
                                          const int64_t* rows, const uint32_t* unsorted_dev,
                                          int64_t n_ids, uint64_t* out_codes,
                                          const int64_t* rank_values, int64_t* out_values,
                                          int32_t* out_values32, uint32_t* err_dev,
                                          void* stream) {
  if (!pairs) return BSB_EINVAL;
  return bs_lookup_rows_impl(col, rows, pairs, unsorted_dev, n_ids, out_codes, rank_values,
                             out_values, out_values32, err_dev, stream);
}

extern "C" int bsb_vbs_lookup_rows(const bsb_vbs* col, const int64_t* rows, int64_t n_ids,
                                   uint64_t* out_padded, const uint64_t* sorted_padded,
                                   const int64_t* dict_values, int64_t n_dict,
                                   int64_t* out_values, int32_t* out_values32,
                                   uint64_t* level_counts, uint32_t* err_dev, void* stream) {
  if (!col || n_ids < 0 || (n_ids > 0 && !rows)) return BSB_EINVAL;
  if (sorted_padded && (!dict_values || n_dict <= 0)) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  if (level_counts) BSB_CUDA(cudaMemsetAsync(level_counts, 0, 8 * kMaxLevels, s));
  if (n_ids == 0) return BSB_OK;
  VbsLookupDesc d;
  fill_lookup_desc(d, col);
  unsigned int* err = err_dev;
  if (!err) {
    const int rc = alloc_err(&err, s);
    if (rc) return rc;
  }
  vbs_lookup_kernel<<<grid_for_l(n_ids, 256), 256, 0, s>>>(d, rows, n_ids, out_padded,
                                                           sorted_padded, dict_values, n_dict,
                                                           out_values, out_values32, err,
                                                           reinterpret_cast<unsigned long long*>(level_counts));
  BSB_LAUNCH_CHECK();
  return err_dev ? BSB_OK : read_err(err, s);
}

extern "C" int bsb_bits_to_rows(const uint32_t* words, int64_t n_rows, int64_t* rows_out,
                                int64_t* n_out_host, void* stream) {
  if (!words || n_rows <= 0 || !n_out_host) return BSB_EINVAL;
  return bits_to_rows_impl(words, n_rows, 0, nullptr, rows_out, nullptr, n_out_host,
                           as_stream(stream));
}

extern "C" int bsb_bits_to_rows_async(const uint32_t* words, int64_t n_rows, int64_t row_offset,
                                      int64_t* rows_out, uint64_t* n_out_dev, void* stream) {
  if (!words || n_rows <= 0) return BSB_EINVAL;
  return bits_to_rows_impl(words, n_rows, row_offset, nullptr, rows_out, n_out_dev, nullptr,
                           as_stream(stream));
}
extern "C" int bsb_bits_to_rows_at(const uint32_t* words, int64_t n_rows, int64_t row_offset,
                                   const int64_t* base_dev, int64_t* rows_out,
                                   uint64_t* n_out_dev, void* stream) {
  if (!words || n_rows <= 0 || !base_dev || !rows_out) return BSB_EINVAL;
  return bits_to_rows_impl(words, n_rows, row_offset, base_dev, rows_out, n_out_dev, nullptr,
                           as_stream(stream));
}

extern "C" int bsb_bits_combine(int32_t op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                                int64_t n_rows, void* stream) {
  if (!a || !out || n_rows < 0 || op < 0 || op > 3 || (op != 2 && !b)) return BSB_EINVAL;
  const int64_t nb = (n_rows + 31) / 32;
  if (nb == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  combine_kernel<<<grid_for_l(nb, 256), 256, 0, s>>>(op, a, b, out, n_rows, nb);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

extern "C" int bsb_bits_popcount(const uint32_t* words, int64_t n_rows, uint64_t* count,
                                 void* stream) {
  if (!words || !count || n_rows < 0) return BSB_EINVAL;
  const int64_t nb = (n_rows + 31) / 32;
  cudaStream_t s = as_stream(stream);
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  if (nb == 0) return BSB_OK;
  popcount_kernel<<<grid_for_l(nb, 256), 256, 0, s>>>(
      words, nb, reinterpret_cast<unsigned long long*>(count));
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

// ===================================================================
// Decoders and fused bitvector-driven lookups
// ===================================================================
namespace bsb {

struct Decoder {
  int kind;
  const int64_t* values;
  const uint64_t* sorted;
  int64_t n;
  const int64_t* e1;
  const int64_t* e2;
};

static void fill_decoder(Decoder& D, const bsb_decode* d) {
  std::memset(&D, 0, sizeof(D));
  if (!d) return;
  D.kind = d->kind;
  D.values = d->values;
  D.sorted = d->sorted_padded;
  D.n = d->n_dict;
  D.e1 = d->e1;
  D.e2 = d->e2;
}

// value of a looked-up code; `code` = right-aligned code (ByteSlice rank or
// PP-VBS code of `len` bytes), `padded` = code << 8*(K-len).  bad is set when
// the code is not in the dictionary.
template <int DK = -1>  // DK >= 0: decoder kind fixed at compile time
__device__ __forceinline__ int64_t decode_value(const Decoder& D, uint64_t code, uint64_t padded,
                                                int len, bool& bad, const int64_t* e1s) {
  switch (DK >= 0 ? DK : D.kind) {
    case 1:
      if (code >= (uint64_t)D.n) {
        bad = true;
        return 0;
      }
      return __ldg(D.values + code);
    case 2: {
      int64_t lo = 0, hi = D.n;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(D.sorted + mid) < padded)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (lo >= D.n || __ldg(D.sorted + lo) != padded) {
        bad = true;
        return 0;
      }
      return __ldg(D.values + lo);
    }
    case 3: {
      // e1 may be a shared-memory copy (e1s); see bsb_decode in the header
      int64_t r = -1;
      const uint32_t b1 = (uint32_t)(code >> (8 * (len - 1))) & 0xFFu;
      const uint64_t n1 = (uint64_t)e1s[b1];
      if (len == 1) {
        const uint32_t r1 = (uint32_t)(n1 >> 32);
        if (r1 != 0xFFFFFFFFu) r = r1;
      } else {
        const uint32_t c = (uint32_t)n1;
        const uint32_t b2 = (uint32_t)(code >> (8 * (len - 2))) & 0xFFu;
        if (c != 0xFFFFFFFFu) {
          const int64_t e = __ldg(D.e2 + 2 * ((int64_t)c * 256 + b2) + (len > 2));
          if (len == 2) {
            r = e;
          } else if (e >= 0 && (int)(e >> 56) == len - 2) {
            const uint64_t sfx = code & ((1ull << (8 * (len - 2))) - 1ull);
            if (sfx >= 1 && sfx <= (uint64_t)((e >> 32) & 0xFFFFFF))
              r = (e & 0xFFFFFFFFll) + (int64_t)sfx - 1;
          }
        }
      }
      if (r < 0) {
        bad = true;
        return 0;
      }
      return __ldg(D.values + r);
    }
    default: return (int64_t)code;
  }
}

// Per-block PP-VBS metadata, loaded once and shared by the block's rows.
struct VbsBlockMeta {
  uint32_t m[kMaxLevels];  // m[j-1] = existence word of level j (j >= 2)
  int64_t dir2;            // sliced: deep-row base of the block
};

__device__ __forceinline__ void vbs_block_meta(const VbsLookupDesc& d, int64_t blk,
                                               VbsBlockMeta& mt) {
#pragma unroll
  for (int j = 2; j <= kMaxLevels; ++j) mt.m[j - 1] = j <= d.K ? __ldg(d.exist[j - 1] + blk) : 0u;
  mt.dir2 = (d.mode != BSB_DEEP_PACKED && d.K >= 2) ? __ldg(d.dir[1] + blk) : 0;
}

// right-aligned code and length of row lr of block blk, given its BS_1 byte
// Code length of row lr from the block's existence words (lengths nest, so
// it is one plus the number of levels >= 2 whose word has the row's bit).
__device__ __forceinline__ int vbs_row_len(const VbsLookupDesc& d, const VbsBlockMeta& mt,
                                           int lr) {
  int L = 1;
#pragma unroll
  for (int j = 2; j <= kMaxLevels; ++j) L += (j <= d.K) ? (int)((mt.m[j - 1] >> lr) & 1u) : 0;
  return L;
}

// Right-aligned code of row lr of block blk, given its BS_1 byte.  All deep
// byte loads are independent (issued together).
template <int MODE = -1>  // MODE >= 0: deep layout fixed at compile time
__device__ __forceinline__ uint64_t vbs_row_code_f(const VbsLookupDesc& d, int64_t blk, int lr,
                                                   const VbsBlockMeta& mt, uint32_t first,
                                                   int& len) {
  const int mode = MODE >= 0 ? MODE : d.mode;
  const uint32_t below = (1u << lr) - 1u;
  len = vbs_row_len(d, mt, lr);
  const int64_t q = mt.dir2 + __popc(mt.m[1] & below);
  uint64_t code = first;
#pragma unroll
  for (int j = 2; j <= kMaxLevels; ++j) {
    if (j > len) continue;  // predicated, not a break: the loads issue together
    uint32_t byte;
    if (mode == BSB_DEEP_SLICED) {
      byte = bp_row_byte(d.deep[j - 1] + (q >> 5) * 32, (int)(q & 31));
    } else {
      byte = __ldg(d.deep[j - 1] + (__ldg(d.dir[j - 1] + blk) + __popc(mt.m[j - 1] & below)));
    }
    code = (code << 8) | byte;
  }
  return code;
}

__device__ __forceinline__ uint64_t vbs_row_code(const VbsLookupDesc& d, int64_t blk, int lr,
                                                 const VbsBlockMeta& mt, int& len) {
  return vbs_row_code_f(d, blk, lr, mt, bp_row_byte(d.bs1 + blk * 32, lr), len);
}


// Fused bitvector -> values.  Warp per tile of 1024 rows.  Lane = block:
// every block with a selected row has its sectors fetched with 256-bit loads
// (ByteSlice: the K plane sectors; PP-VBS: the BS_1 sector) into the warp's
// shared-memory stage, all in flight together, plus (PP-VBS) its existence
// words and level-2 directory entry.  The lane then lists its block's set
// rows as 16-bit records (row in tile | code length - 1), the
// length coming from bit-sliced counts of the nested existence words.  Lane
// k then assembles listed rows k, k+32, ... (kRowsPerLane at a time, their
// deep-byte loads in flight together), decodes them (PPE first-level table
// in shared memory) and writes them contiguously.  A bad code sets *err
// (UINT64_MAX when err is the output count).
constexpr int kBitsThreads = 128;
__device__ uint32_t g_dense_rows = 96;  // selected rows per tile from which deep loads allocate in L1
void set_dense_rows(int64_t v) {
  const uint32_t h = v < 0 ? 96u : (uint32_t)v;
  cudaMemcpyToSymbol(g_dense_rows, &h, 4);
}

// per-warp shared memory: row records (u16) + stage (+ PP-VBS existence words, directory)
__host__ __device__ constexpr int bits_stage_bytes(bool vbs, int K) {
  return vbs ? 2048 + 1024 + 128 * (K > 1 ? K - 1 : 0) + 256 : 2048 + 1024 * K;
}

__device__ __forceinline__ void sts256(uint8_t* dst, const uint32_t (&v)[8]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
  d[0] = make_uint4(v[0], v[1], v[2], v[3]);
  d[1] = make_uint4(v[4], v[5], v[6], v[7]);
}

template <bool VBS, int DK, int MODE, int KT, bool COOP = false>
__global__ void __launch_bounds__(kBitsThreads) lookup_bits_kernel(
    const uint8_t* __restrict__ slices, int64_t stride, int K, int width,  // ByteSlice
    const __grid_constant__ VbsLookupDesc vd,                              // PP-VBS
    const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
    const int64_t* __restrict__ tile_incl, const __grid_constant__ Decoder D,
    uint64_t* __restrict__ oc, int64_t* __restrict__ ov, int32_t* __restrict__ ov32,
    unsigned long long* __restrict__ err, long long* __restrict__ cta_tot) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ long long s_wtot[kBitsThreads / 32 + 1];
  int64_t* e1s = reinterpret_cast<int64_t*>(dsm);  // DK == 3: first-level PPE table
  if (DK == 3) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) e1s[i] = __ldg(D.e1 + i);
    __syncthreads();
  }
  const int KL = KT > 0 ? KT : (VBS ? vd.K : K);
  const int KD = KL > 1 ? KL - 1 : 0;
  uint8_t* wbase = dsm + (DK == 3 ? 2048 : 0) + (threadIdx.x >> 5) * bits_stage_bytes(VBS, KL);
  using Rec = uint16_t;
  constexpr int kRowsPerLane = 1;  // rows assembled per lane at a time (bit-plane sectors: 8 registers per level in flight)
  Rec* idx = reinterpret_cast<Rec*>(wbase);
  uint8_t* stage = wbase + 1024 * sizeof(Rec);
  uint32_t* smeta = reinterpret_cast<uint32_t*>(stage + 1024);  // PACKED: m[(j-2)*32 + b]
  int64_t* sdir = reinterpret_cast<int64_t*>(smeta + 32 * KD);   // level-2 directory
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int shift = VBS ? 0 : 8 * KL - width;
  bool bad = false;
  // Tile order.  cta_tot NULL: tiles round-robin over the warps, the selected
  // rows before a tile come from tile_incl (tile popcount + scan kernels).
  // cta_tot given (small columns, cooperative launch): every warp owns a
  // contiguous run of tiles; the warps count their runs, the CTAs exchange
  // totals across one grid barrier, and the running position is carried
  // through the run -- the whole fused lookup is one kernel.
  int64_t t = warp, t_end = ntiles, step = nwarps, running = 0;
  if (COOP) {
    const int wq = threadIdx.x >> 5;
    const int64_t per_warp = (ntiles + nwarps - 1) / nwarps;
    t = warp * per_warp;
    t_end = t + per_warp < ntiles ? t + per_warp : ntiles;
    step = 1;
    uint32_t c1 = 0;
    for (int64_t q = t; q < t_end; ++q)
      if (q * 32 + lane < nb) c1 += __popc(__ldg(words + q * 32 + lane));
    c1 = __reduce_add_sync(kFull, c1);
    if (lane == 0) s_wtot[wq] = c1;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long sum = 0;
      for (int q = 0; q < kBitsThreads / 32; ++q) sum += s_wtot[q];
      cta_tot[blockIdx.x] = sum;
      if (blockIdx.x == 0) *err = 0ull;  // the count (atomicMax below; ~0 after a bad code)
    }
    cooperative_groups::this_grid().sync();
    if (wq == 0) {
      long long before = 0, grand = 0;
      for (unsigned i = lane; i < gridDim.x; i += 32) {
        const long long v = __ldcg(cta_tot + i);
        grand += v;
        if (i < blockIdx.x) before += v;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        before += __shfl_xor_sync(kFull, before, d);
        grand += __shfl_xor_sync(kFull, grand, d);
      }
      if (lane == 0) {
        s_wtot[kBitsThreads / 32] = before;
        if (blockIdx.x == 0) atomicMax(err, (unsigned long long)grand);
      }
    }
    __syncthreads();
    running = s_wtot[kBitsThreads / 32];
    for (int q = 0; q < wq; ++q) running += s_wtot[q];
  }
  if (!COOP) {  // the compiler keeps ntiles / nwarps, no extra registers
    t_end = ntiles;
    step = nwarps;
  }
  uint32_t w = 0;
  if (t < t_end) w = (t * 32 + lane) < nb ? __ldg(words + t * 32 + lane) : 0u;
  for (; t < t_end; t += step) {
    const int64_t tn = t + step;
    const uint32_t wn = (tn < t_end && tn * 32 + lane < nb) ? __ldg(words + tn * 32 + lane) : 0u;
    const uint32_t c = __popc(w);
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (total) {
      const int64_t blk = t * 32 + lane;
      uint32_t m[kMaxLevels + 1];
#pragma unroll
      for (int j = 0; j <= kMaxLevels; ++j) m[j] = 0u;
      if (VBS) {
        const bool in = blk < nb;
        if (w) {
          // deeper words only matter when a selected row owns a level-2 byte
          m[2] = (in && KL >= 2) ? __ldg(vd.exist[1] + blk) : 0u;
          const bool deep = (m[2] & w) != 0u;
#pragma unroll
          for (int j = 3; j <= kMaxLevels; ++j)
            if (j <= KL) m[j] = (in && deep) ? __ldg(vd.exist[j - 1] + blk) : 0u;
          sdir[lane] = (in && deep && MODE != BSB_DEEP_PACKED) ? __ldg(vd.dir[1] + blk) : 0;
          uint32_t v[8];
          ldg256_free(vd.bs1 + blk * 32, v);
          sts256(stage + lane * 32, v);
          if (KL >= 2) smeta[lane] = m[2];  // the rows' deep-row offsets: popc(M_2 & below)
          if (MODE == BSB_DEEP_PACKED) {
#pragma unroll
            for (int j = 3; j <= kMaxLevels; ++j)
              if (j <= KL) smeta[(j - 2) * 32 + lane] = m[j];
          }
        }
      } else if (w) {
        if (KT > 0) {
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            uint32_t v[8];
            ldg256_free(slices + j * stride + blk * 32, v);
            sts256(stage + j * 1024 + lane * 32, v);
          }
        } else {  // run-time slice count: a plain loop (the unrolled, predicated form
                  // measured 40 % slower with the rank-table decode)
          for (int j = 0; j < K; ++j) {
            uint32_t v[8];
            ldg256_free(slices + j * stride + blk * 32, v);
            sts256(stage + j * 1024 + lane * 32, v);
          }
        }
      }
      const uint32_t excl = incl - c;
      const int64_t tbase = COOP ? running : (t ? __ldg(tile_incl + t - 1) : 0);
      // each lane lists its block's set rows (ascending) as records
      {
        // bit-sliced (code length - 1) of the block's rows; lengths nest, so
        // length - 1 >= k iff the row is in M_{k+1}
        const uint32_t c0 = (m[2] & ~m[3]) | (m[4] & ~m[5]) | (m[6] & ~m[7]) | m[8];
        const uint32_t c1 = (m[3] & ~m[5]) | m[7];
        const uint32_t c2 = m[5];
        uint32_t rest = w;
        uint32_t o = excl;
        while (rest) {
          const int bit = __ffs(rest) - 1;
          rest &= rest - 1;
          uint32_t rec = (uint32_t)((lane << 5) | bit);
          if (VBS) {
            const uint32_t lm1 = ((c0 >> bit) & 1u) | (((c1 >> bit) & 1u) << 1) |
                                 (((c2 >> bit) & 1u) << 2);
            rec |= lm1 << 10;
          }
          idx[o++] = (Rec)rec;
        }
      }
      __syncwarp();
      const bool dense = total >= g_dense_rows;
      for (uint32_t k0 = lane; k0 < total; k0 += 32 * kRowsPerLane) {
        uint64_t code[kRowsPerLane], pad[kRowsPerLane];
        int len[kRowsPerLane];
        bool on[kRowsPerLane];
#pragma unroll
        for (int u = 0; u < kRowsPerLane; ++u) {
          const uint32_t k = k0 + 32 * u;
          on[u] = k < total;
          const uint32_t r = on[u] ? idx[k] : 0u;
          const int bl = (int)((r >> 5) & 31);
          const int lr = (int)(r & 31);
          if (VBS) {
            len[u] = on[u] ? 1 + (int)((r >> 10) & 7u) : 1;
            uint64_t cd = bp_row_byte_smem(stage + bl * 32, lr);
            const uint32_t below = (1u << lr) - 1u;
            const int64_t q = MODE == BSB_DEEP_PACKED || len[u] < 2
                                  ? 0 : sdir[bl] + __popc(smeta[bl] & below);
            const int64_t blkr = t * 32 + bl;
#pragma unroll
            for (int j = 2; j <= kMaxLevels; ++j) {
              if (j <= KL && j <= len[u]) {
                uint32_t byte;
                if (MODE == BSB_DEEP_SLICED) {
                  // a dense tile's rows share deep sectors: let L1 keep them
                  const uint8_t* sp = vd.deep[j - 1] + (q >> 5) * 32;
                  byte = dense ? bp_row_byte_l1(sp, (int)(q & 31))
                               : bp_row_byte(sp, (int)(q & 31));
                } else {
                  byte = __ldg(vd.deep[j - 1] + (__ldg(vd.dir[j - 1] + blkr) +
                                                 __popc(smeta[(j - 2) * 32 + bl] & below)));
                }
                cd = (cd << 8) | byte;
              }
            }
            code[u] = cd;
            pad[u] = cd << (8 * (KL - len[u]));
          } else {
            uint64_t cd = 0;
#pragma unroll
            for (int j = 0; j < kMaxLevels; ++j)
              if (j < (KT > 0 ? KT : K)) cd = (cd << 8) | bp_row_byte_smem(stage + j * 1024 + bl * 32, lr);
            code[u] = pad[u] = cd >> shift;
            len[u] = 0;
          }
        }
#pragma unroll
        for (int u = 0; u < kRowsPerLane; ++u) {
          if (!on[u]) continue;
          const int64_t v = decode_value<DK>(D, code[u], pad[u], len[u], bad,
                                             DK == 3 ? e1s : D.e1);
          emit(oc, ov, ov32, tbase + k0 + 32 * u, pad[u], v);
        }
      }
      __syncwarp();
    }
    if (COOP) running += total;
    w = wn;
  }
  if (bad) {
    if (COOP) atomicMax(err, ~0ull); else *err = ~0ull;
  }
}

// Row-id lookup + general decode; kVbsIds ids per thread in flight.
template <int MODE, bool PAIRS>
__global__ void vbs_lookup_rows_dec_kernel(const __grid_constant__ VbsLookupDesc vd,
                                           const void* __restrict__ rows, int64_t n_ids,
                                           const __grid_constant__ Decoder D,
                                           uint64_t* __restrict__ oc, int64_t* __restrict__ ov,
                                           int32_t* __restrict__ ov32,
                                           unsigned int* __restrict__ err,
                                           const uint32_t* __restrict__ gate, bool want) {
  __shared__ int64_t e1sm[256];
  if (gate_closed(gate, want)) return;
  const int64_t* e1s = D.e1;
  if (D.kind == 3) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) e1sm[i] = __ldg(D.e1 + i);
    __syncthreads();
    e1s = e1sm;
  }
  bool bad = false, oob = false;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n_ids;
       i0 += nthr * kVbsIds) {
    uint64_t code[kVbsIds];
    int len[kVbsIds];
#pragma unroll
    for (int u = 0; u < kVbsIds; ++u) {
      const int64_t i = i0 + u * nthr;
      int64_t r = i < n_ids ? id_at<PAIRS>(rows, i) : 0;
      if ((uint64_t)r >= (uint64_t)vd.n_rows) {  // IndexError in the reference; never read it
        oob = true;
        r = 0;
      }
      const int64_t blk = r >> 5;
      const int lr = (int)(r & 31);
      const uint32_t first = bp_row_byte(vd.bs1 + blk * 32, lr);
      // a row outside M_2 has a 1-byte code: no deeper existence words,
      // directory entry or deep bytes to fetch
      const uint32_t m2 = vd.K >= 2 ? __ldg(vd.exist[1] + blk) : 0u;
      if (!((m2 >> lr) & 1u)) {
        code[u] = first;
        len[u] = 1;
      } else {
        VbsBlockMeta mt;
        mt.m[0] = 0u;
        mt.m[1] = m2;
#pragma unroll
        for (int j = 3; j <= kMaxLevels; ++j) mt.m[j - 1] = j <= vd.K ? __ldg(vd.exist[j - 1] + blk) : 0u;
        mt.dir2 = MODE != BSB_DEEP_PACKED ? __ldg(vd.dir[1] + blk) : 0;
        code[u] = vbs_row_code_f<MODE>(vd, blk, lr, mt, first, len[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kVbsIds; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i >= n_ids) break;
      const uint64_t padded = code[u] << (8 * (vd.K - len[u]));
      const int64_t v = decode_value(D, code[u], padded, len[u], bad, e1s);
      emit(oc, ov, ov32, i, padded, v);
    }
  }
  if (bad) atomicOr(err, kErrNotFound);
  if (__any_sync(kFull, oob) && (threadIdx.x & 31) == 0) atomicOr(err, kErrIndex);
}



// Columns of at most this many 1024-row tiles take the one-kernel cooperative
// fused lookup (bsb_tune "coop_tiles"; 0 = never).  Measured (B200, 1 % / 20 %
// selections): 2^24 rows 34 -> 22 us / 49 -> 49 us (ByteSlice), 34 -> 27 / 80
// -> 80 us (PP-VBS); 2^26 rows 59 -> 53 / 137 -> 133 and 86 -> 82 / 273 ->
// 291 us: the launches it saves stop mattering and the contiguous tile runs
// cost the dense PP-VBS case, hence 2^14 tiles.
static int64_t g_coop_tiles = 1 << 14;
void set_coop_tiles(int64_t v) { g_coop_tiles = v < 0 ? (1 << 14) : v; }
static bool coop_lookup_ok(int64_t ntiles) {
  static int supported = [] {
    int dev = 0, ok = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
    return ok;
  }();
  return supported && ntiles <= g_coop_tiles;
}

template <bool VBS>
static int lookup_bits_impl(const bsb_byteslice* bcol, const bsb_vbs* vcol,
                            const uint32_t* words, const bsb_decode* dec, uint64_t* oc,
                            int64_t* ov, int32_t* ov32, uint64_t* n_out_dev, cudaStream_t s) {
  const int64_t n = VBS ? vcol->n_rows : bcol->n_rows;
  const int64_t nb = (n + 31) / 32;
  const int64_t ntiles = (nb + 31) / 32;
  // Small selections' columns (<= kCoopTiles tiles): ONE cooperative kernel
  // (the tile popcount / scan / copy launches cost more than the lookup).
  const bool coop = coop_lookup_ok(ntiles);
  const int64_t cta_cap = (int64_t)sm_count() * 32;
  int64_t* tc = nullptr;
  BSB_CUDA(cudaMallocAsync(&tc, (coop ? cta_cap + 4 : ntiles * 2 + 4) * sizeof(int64_t), s));
  int64_t* incl = coop ? nullptr : tc + ntiles + 1;
  unsigned long long* errw =
      reinterpret_cast<unsigned long long*>(coop ? tc + cta_cap + 1 : incl + ntiles + 1);
  void* tmp = nullptr;
  if (!coop) {
    launch_tile_popc(words, nb, ntiles, tc, s);
    BSB_LAUNCH_CHECK();
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, tc, incl, ntiles, s);
    BSB_CUDA(cudaMallocAsync(&tmp, tb + 16, s));
    cub::DeviceScan::InclusiveSum(tmp, tb, tc, incl, ntiles, s);
    BSB_LAUNCH_CHECK();
    if (n_out_dev)
      BSB_CUDA(cudaMemcpyAsync(n_out_dev, incl + ntiles - 1, 8, cudaMemcpyDeviceToDevice, s));
    else
      BSB_CUDA(cudaMemsetAsync(errw, 0, 8, s));
  }
  Decoder D;
  fill_decoder(D, dec);
  VbsLookupDesc vd;
  std::memset(&vd, 0, sizeof(vd));
  if (VBS) fill_lookup_desc(vd, vcol);
  const int wpb = kBitsThreads / 32;
  const int smem = wpb * bits_stage_bytes(VBS, VBS ? vcol->max_len : bcol->n_slices) +
                   (D.kind == 3 ? 2048 : 0);
  auto launch1 = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      BSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    BSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBitsThreads, smem));
    const int bgrid = (int)std::min<int64_t>((ntiles + wpb - 1) / wpb,
                                             (int64_t)sm_count() * (per_sm < 1 ? 1 : per_sm));
    unsigned long long* nout = n_out_dev ? reinterpret_cast<unsigned long long*>(n_out_dev) : errw;
    if (coop) {
      const uint8_t* a_sl = VBS ? nullptr : bcol->slices;
      int64_t a_stride = VBS ? 0 : bcol->stride;
      int a_k = VBS ? 0 : bcol->n_slices, a_w = VBS ? 0 : bcol->width_bits;
      int64_t a_nb = nb, a_nt = ntiles;
      const int64_t* a_incl = nullptr;
      long long* a_cta = reinterpret_cast<long long*>(tc);
      void* args[] = {&a_sl, &a_stride, &a_k, &a_w, &vd, &words, &a_nb, &a_nt, &a_incl,
                      &D, &oc, &ov, &ov32, &nout, &a_cta};
      BSB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern),
                                           dim3(bgrid < 1 ? 1 : bgrid), dim3(kBitsThreads), args,
                                           (size_t)smem, s));
      return BSB_OK;
    }
    kern<<<bgrid < 1 ? 1 : bgrid, kBitsThreads, smem, s>>>(
        VBS ? nullptr : bcol->slices, VBS ? 0 : bcol->stride, VBS ? 0 : bcol->n_slices,
        VBS ? 0 : bcol->width_bits, vd, words, nb, ntiles, incl, D, oc, ov, ov32, nout, nullptr);
    BSB_LAUNCH_CHECK();
    return BSB_OK;
  };
#define BSB_LB(...) \
  (coop ? launch1(lookup_bits_kernel<__VA_ARGS__, true>) : launch1(lookup_bits_kernel<__VA_ARGS__, false>))
  int rc;
  if (!VBS) {
    // ByteSlice: the common slice counts as a template argument (no dead
    // level iterations in the per-row assembly)
    auto bs_k = [&](auto dk) -> int {
      constexpr int DKC = decltype(dk)::value;
      switch (bcol->n_slices) {
        case 2: return BSB_LB(VBS, DKC, 0, 2);
        case 3: return BSB_LB(VBS, DKC, 0, 3);
        case 4: return BSB_LB(VBS, DKC, 0, 4);
        default: return BSB_LB(VBS, DKC, 0, 0);
      }
    };
    // (with the rank-table decode the templated form's 48 registers cost more
    // occupancy than the dead iterations: cfg4 z24 243 -> 354 us; run-time K)
    rc = D.kind == 1 ? BSB_LB(VBS, 1, 0, 0) : bs_k(std::integral_constant<int, 0>());
  } else {
    // SLICED (the default deep layout) gets the code length as a template
    // argument; the other layouts take it at run time.
    auto sliced_k = [&](auto dk) -> int {
      constexpr int DKC = decltype(dk)::value;
      switch (vcol->max_len) {
        case 2: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 2);
        case 3: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 3);
        case 4: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 4);
        case 5: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 5);
        case 6: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 6);
        case 7: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 7);
        case 8: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 8);
        default: return BSB_LB(VBS, DKC, BSB_DEEP_SLICED, 0);
      }
    };
    auto by_mode = [&](auto dk) -> int {
      constexpr int DKC = decltype(dk)::value;
      switch (vcol->deep_mode) {
        case BSB_DEEP_PACKED: return BSB_LB(VBS, DKC, BSB_DEEP_PACKED, 0);
        default: return sliced_k(dk);
      }
    };
    switch (D.kind) {
      case 0: rc = by_mode(std::integral_constant<int, 0>()); break;
      case 2: rc = by_mode(std::integral_constant<int, 2>()); break;
      default: rc = by_mode(std::integral_constant<int, 3>()); break;
    }
  }
#undef BSB_LB
  if (rc != BSB_OK) return rc;
  if (tmp) BSB_CUDA(cudaFreeAsync(tmp, s));
  if (n_out_dev || D.kind == 0) {
    BSB_CUDA(cudaFreeAsync(tc, s));
    return BSB_OK;
  }
  unsigned long long h = 0;  // cooperative form: the count, or ~0 after a bad code
  BSB_CUDA(cudaMemcpyAsync(&h, errw, 8, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(tc, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (coop ? h == ~0ull : h != 0) {
    set_error_msg("code not in dictionary");
    return BSB_ENOTFOUND;
  }
  return BSB_OK;
}

}  // namespace bsb

extern "C" int bsb_byteslice_lookup_bits(const bsb_byteslice* col, const uint32_t* words,
                                         const bsb_decode* dec, uint64_t* out_codes,
                                         int64_t* out_values, int32_t* out_values32,
                                         uint64_t* n_out_dev, void* stream) {
  if (!col || !words || col->n_rows <= 0) return BSB_EINVAL;
  if (dec && dec->kind != 0 && dec->kind != 1) return BSB_EINVAL;
  return lookup_bits_impl<false>(col, nullptr, words, dec, out_codes, out_values, out_values32,
                                 n_out_dev, as_stream(stream));
}

extern "C" int bsb_vbs_lookup_bits(const bsb_vbs* col, const uint32_t* words,
                                   const bsb_decode* dec, uint64_t* out_padded,
                                   int64_t* out_values, int32_t* out_values32,
                                   uint64_t* n_out_dev, void* stream) {
  if (!col || !words || col->n_rows <= 0) return BSB_EINVAL;
  if (dec && (dec->kind == 1 || dec->kind > 3)) return BSB_EINVAL;
  return lookup_bits_impl<true>(nullptr, col, words, dec, out_padded, out_values, out_values32,
                                n_out_dev, as_stream(stream));
}

// pairs / unsorted_dev: see bs_lookup_rows_impl
static int vbs_lookup_rows_dec_impl(const bsb_vbs* col, const int64_t* rows,
                                    const uint64_t* pairs, const uint32_t* unsorted_dev,
                                    int64_t n_ids, const bsb_decode* dec, uint64_t* out_padded,
                                    int64_t* out_values, int32_t* out_values32,
                                    uint32_t* err_dev, void* stream, bool automatic = false) {
  if (!col || n_ids < 0 || (n_ids > 0 && !rows && !pairs)) return BSB_EINVAL;
  if (pairs && unsorted_dev && !rows) return BSB_EINVAL;
  if (dec && (dec->kind == 1 || dec->kind > 3)) return BSB_EINVAL;
  if (col->deep_mode != BSB_DEEP_PACKED && col->deep_mode != BSB_DEEP_SLICED) return BSB_EINVAL;
  if (n_ids == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  Decoder D;
  fill_decoder(D, dec);
  VbsLookupDesc vd;
  fill_lookup_desc(vd, col);
  const cudaStream_t ps = s;
  unsigned int* err = err_dev;
  AutoScratch au;
  automatic = automatic && auto_fits(n_ids, col->n_rows);
  const int polled = automatic ? rows_order_poll(rows, n_ids, s) : -1;  // see bs_lookup_rows_impl
  if (polled == 0) automatic = false;
  if (automatic) {
    const int rc = auto_begin(au, rows, n_ids, &err, s, polled < 0);
    if (rc) return rc;
    pairs = au.pairs;
    unsorted_dev = polled < 0 ? au.unsorted : nullptr;
  } else if (!err) {
    BSB_CUDA(cudaMallocAsync(&err, 4, s));
    BSB_CUDA(cudaMemsetAsync(err, 0, 4, s));
  }
  const int g = grid_for_l((n_ids + kVbsIds - 1) / kVbsIds, 256);
  const bool sliced = col->deep_mode == BSB_DEEP_SLICED;
  if (!pairs || unsorted_dev) {
    const uint32_t* gate = pairs ? unsorted_dev : nullptr;
    if (sliced)
      vbs_lookup_rows_dec_kernel<BSB_DEEP_SLICED, false><<<g, 256, 0, s>>>(
          vd, rows, n_ids, D, out_padded, out_values, out_values32, err, gate, false);
    else
      vbs_lookup_rows_dec_kernel<BSB_DEEP_PACKED, false><<<g, 256, 0, s>>>(
          vd, rows, n_ids, D, out_padded, out_values, out_values32, err, gate, false);
    BSB_LAUNCH_CHECK();
  }
  if (automatic) {
    const int rc = rows_bucket_gated(rows, n_ids, col->n_rows, au.pairs, unsorted_dev, ps);
    if (rc) return rc;
  }
  if (pairs) {
    PairOut t;
    int rc = pair_out_alloc(t, n_ids, out_padded, out_values, out_values32, ps);
    if (rc) return rc;
    if (sliced)
      vbs_lookup_rows_dec_kernel<BSB_DEEP_SLICED, true><<<g, 256, 0, ps>>>(
          vd, pairs, n_ids, D, t.oc, t.ov, t.ov32, err, unsorted_dev, true);
    else
      vbs_lookup_rows_dec_kernel<BSB_DEEP_PACKED, true><<<g, 256, 0, ps>>>(
          vd, pairs, n_ids, D, t.oc, t.ov, t.ov32, err, unsorted_dev, true);
    BSB_LAUNCH_CHECK();
    rc = pair_out_scatter(t, pairs, n_ids, out_padded, out_values, out_values32, unsorted_dev,
                          ps);
    if (rc) return rc;
  }
  if (automatic) return auto_end(au, err, !err_dev, s);
  if (err_dev) return BSB_OK;
  return read_err(err, s);
}

extern "C" int bsb_vbs_lookup_rows_dec_auto(const bsb_vbs* col, const int64_t* rows,
                                            int64_t n_ids, const bsb_decode* dec,
                                            uint64_t* out_padded, int64_t* out_values,
                                            int32_t* out_values32, uint32_t* err_dev,
                                            void* stream) {
  if (!rows && n_ids > 0) return BSB_EINVAL;
  return vbs_lookup_rows_dec_impl(col, rows, nullptr, nullptr, n_ids, dec, out_padded,
                                  out_values, out_values32, err_dev, stream, true);
}

extern "C" int bsb_vbs_lookup_rows_dec(const bsb_vbs* col, const int64_t* rows, int64_t n_ids,
                                       const bsb_decode* dec, uint64_t* out_padded,
                                       int64_t* out_values, int32_t* out_values32,
                                       uint32_t* err_dev, void* stream) {
  return vbs_lookup_rows_dec_impl(col, rows, nullptr, nullptr, n_ids, dec, out_padded,
                                  out_values, out_values32, err_dev, stream);
}

extern "C" int bsb_vbs_lookup_pairs_dec(const bsb_vbs* col, const uint64_t* pairs,
                                        const int64_t* rows, const uint32_t* unsorted_dev,
                                        int64_t n_ids, const bsb_decode* dec,
                                        uint64_t* out_padded, int64_t* out_values,
                                        int32_t* out_values32, uint32_t* err_dev, void* stream) {
  if (!pairs) return BSB_EINVAL;
  return vbs_lookup_rows_dec_impl(col, rows, pairs, unsorted_dev, n_ids, dec, out_padded,
                                  out_values, out_values32, err_dev, stream);
}
