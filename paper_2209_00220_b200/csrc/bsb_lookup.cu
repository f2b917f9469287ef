// bsb_lookup.cu -- row lookups (ByteSlice / PP-VBS), decode, bitvector
// compaction and word-level bitvector algebra.
#include <cub/device/device_scan.cuh>

#include <cstring>

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

__global__ void bs_lookup_kernel(const uint8_t* __restrict__ slices, int64_t stride, int K,
                                 int width, const int64_t* __restrict__ rows, int64_t n_ids,
                                 uint64_t* __restrict__ out_codes,
                                 const int64_t* __restrict__ rank_values,
                                 int64_t* __restrict__ out_values,
                                 int32_t* __restrict__ out_values32) {
  const int shift = 8 * K - width;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n_ids;
       i0 += nthr * kIdsPerThread) {
    int64_t pos[kIdsPerThread];
    uint64_t c[kIdsPerThread];
#pragma unroll
    for (int u = 0; u < kIdsPerThread; ++u) {
      const int64_t i = i0 + u * nthr;
      const int64_t r = i < n_ids ? __ldg(rows + i) : 0;
      pos[u] = (r & ~int64_t(31)) + swz((int)(r & 31));
      c[u] = 0;
    }
    for (int j = 0; j < K; ++j) {
#pragma unroll
      for (int u = 0; u < kIdsPerThread; ++u)
        if (i0 + u * nthr < n_ids)
          c[u] = (c[u] << 8) | __ldg(slices + (int64_t)j * stride + pos[u]);
    }
#pragma unroll
    for (int u = 0; u < kIdsPerThread; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i >= n_ids) break;
      const uint64_t cd = c[u] >> shift;
      if (out_codes) out_codes[i] = cd;
      if (rank_values) {
        const int64_t v = __ldg(rank_values + cd);
        if (out_values) out_values[i] = v;
        if (out_values32) out_values32[i] = (int32_t)v;
      }
    }
  }
}

struct VbsLookupDesc {
  const uint8_t* bs1;
  const uint8_t* deep[kMaxLevels];
  const uint32_t* exist[kMaxLevels];
  const int64_t* dir[kMaxLevels];
  int K;
  int mode;
};

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
    const int64_t r = __ldg(rows + i);
    const int64_t b = r >> 5;
    const int lr = (int)(r & 31);
    uint64_t code = (uint64_t)__ldg(d.bs1 + (b * 32 + swz(lr))) << (8 * (K - 1));
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
        byte = __ldg(d.deep[j - 1] + ((pos2 & ~int64_t(31)) + swz((int)(pos2 & 31))));
      } else if (d.mode == BSB_DEEP_PLANES) {
        const uint16_t v = __ldg(reinterpret_cast<const uint16_t*>(d.deep[((j - 2) >> 1) + 1]) + pos2);
        byte = ((j - 2) & 1) ? (v & 0xFFu) : (v >> 8);
      } else {
        const int64_t pos = d.mode == BSB_DEEP_RANK2 ? pos2
                                                     : __ldg(d.dir[j - 1] + b) + __popc(w & below);
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
        atomicOr(err, 1u);
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
__global__ void tile_popc_kernel(const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
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

__global__ void tile_emit_kernel(const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
                                 const int64_t* __restrict__ tile_incl, int64_t row_offset,
                                 int64_t* __restrict__ rows_out) {
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
                             int64_t* rows_out, uint64_t* n_out_dev, int64_t* n_out_host,
                             cudaStream_t s) {
  const int64_t nb = (n_rows + 31) / 32;
  const int64_t ntiles = (nb + 31) / 32;
  int64_t* tc = nullptr;
  BSB_CUDA(cudaMallocAsync(&tc, (ntiles * 2 + 2) * sizeof(int64_t), s));
  int64_t* incl = tc + ntiles + 1;
  const int grid = grid_for_l(ntiles * 32, 256);
  tile_popc_kernel<<<grid, 256, 0, s>>>(words, nb, ntiles, tc);
  BSB_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, tc, incl, ntiles, s);
  void* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, tc, incl, ntiles, s);
  BSB_LAUNCH_CHECK();
  if (rows_out) {
    tile_emit_kernel<<<grid, 256, 0, s>>>(words, nb, ntiles, incl, row_offset, rows_out);
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

extern "C" int bsb_byteslice_lookup_rows(const bsb_byteslice* col, const int64_t* rows,
                                         int64_t n_ids, uint64_t* out_codes,
                                         const int64_t* rank_values, int64_t* out_values,
                                         int32_t* out_values32, void* stream) {
  if (!col || n_ids < 0 || (n_ids > 0 && !rows)) return BSB_EINVAL;
  if (n_ids == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  bs_lookup_kernel<<<grid_for_l((n_ids + kIdsPerThread - 1) / kIdsPerThread, 256), 256, 0, s>>>(
      col->slices, col->stride, col->n_slices, col->width_bits, rows, n_ids, out_codes,
      rank_values, out_values, out_values32);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

extern "C" int bsb_vbs_lookup_rows(const bsb_vbs* col, const int64_t* rows, int64_t n_ids,
                                   uint64_t* out_padded, const uint64_t* sorted_padded,
                                   const int64_t* dict_values, int64_t n_dict,
                                   int64_t* out_values, int32_t* out_values32,
                                   uint64_t* level_counts, void* stream) {
  if (!col || n_ids < 0 || (n_ids > 0 && !rows)) return BSB_EINVAL;
  if (sorted_padded && (!dict_values || n_dict <= 0)) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  if (level_counts) BSB_CUDA(cudaMemsetAsync(level_counts, 0, 8 * kMaxLevels, s));
  if (n_ids == 0) return BSB_OK;
  VbsLookupDesc d;
  std::memset(&d, 0, sizeof(d));
  d.bs1 = col->bs1;
  d.K = col->max_len;
  d.mode = col->deep_mode;
  for (int j = 0; j < kMaxLevels; ++j) {
    d.deep[j] = col->deep[j];
    d.exist[j] = col->exist[j];
    d.dir[j] = col->block_dir[j];
  }
  unsigned int* err = nullptr;
  if (sorted_padded) {
    BSB_CUDA(cudaMallocAsync(&err, 4, s));
    BSB_CUDA(cudaMemsetAsync(err, 0, 4, s));
  }
  vbs_lookup_kernel<<<grid_for_l(n_ids, 256), 256, 0, s>>>(d, rows, n_ids, out_padded,
                                                           sorted_padded, dict_values, n_dict,
                                                           out_values, out_values32, err,
                                                           reinterpret_cast<unsigned long long*>(level_counts));
  BSB_LAUNCH_CHECK();
  if (sorted_padded) {
    unsigned int h = 0;
    BSB_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s));
    BSB_CUDA(cudaFreeAsync(err, s));
    BSB_CUDA(cudaStreamSynchronize(s));
    if (h) {
      set_error_msg("padded code not in dictionary");
      return BSB_ENOTFOUND;
    }
  }
  return BSB_OK;
}

extern "C" int bsb_bits_to_rows(const uint32_t* words, int64_t n_rows, int64_t* rows_out,
                                int64_t* n_out_host, void* stream) {
  if (!words || n_rows <= 0 || !n_out_host) return BSB_EINVAL;
  return bits_to_rows_impl(words, n_rows, 0, rows_out, nullptr, n_out_host, as_stream(stream));
}

extern "C" int bsb_bits_to_rows_async(const uint32_t* words, int64_t n_rows, int64_t row_offset,
                                      int64_t* rows_out, uint64_t* n_out_dev, void* stream) {
  if (!words || n_rows <= 0) return BSB_EINVAL;
  return bits_to_rows_impl(words, n_rows, row_offset, rows_out, n_out_dev, nullptr,
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
  const int32_t* t1;
  const int32_t* c1;
  const int32_t* t2;
  const int32_t* c2;
  const int64_t* leaf_start;
  const int32_t* leaf_size;
  const int32_t* leaf_beta;
};

static void fill_decoder(Decoder& D, const bsb_decode* d) {
  std::memset(&D, 0, sizeof(D));
  if (!d) return;
  D.kind = d->kind;
  D.values = d->values;
  D.sorted = d->sorted_padded;
  D.n = d->n_dict;
  D.t1 = d->t1;
  D.c1 = d->c1;
  D.t2 = d->t2;
  D.c2 = d->c2;
  D.leaf_start = d->leaf_start;
  D.leaf_size = d->leaf_size;
  D.leaf_beta = d->leaf_beta;
}

// value of a looked-up code; `code` = right-aligned code (ByteSlice rank or
// PP-VBS code of `len` bytes), `padded` = code << 8*(K-len).  bad is set when
// the code is not in the dictionary.
template <int DK = -1>  // DK >= 0: decoder kind fixed at compile time
__device__ __forceinline__ int64_t decode_value(const Decoder& D, uint64_t code, uint64_t padded,
                                                int len, bool& bad) {
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
      int32_t r = -1;
      const uint32_t b1 = (uint32_t)(code >> (8 * (len - 1))) & 0xFFu;
      if (len == 1) {
        r = __ldg(D.t1 + b1);
      } else {
        const int32_t c = __ldg(D.c1 + b1);
        const uint32_t b2 = (uint32_t)(code >> (8 * (len - 2))) & 0xFFu;
        if (c >= 0) {
          if (len == 2) {
            r = __ldg(D.t2 + (int64_t)c * 256 + b2);
          } else {
            const int32_t lf = __ldg(D.c2 + (int64_t)c * 256 + b2);
            if (lf >= 0 && __ldg(D.leaf_beta + lf) == len - 2) {
              const uint64_t sfx = code & ((1ull << (8 * (len - 2))) - 1ull);
              if (sfx >= 1 && sfx <= (uint64_t)__ldg(D.leaf_size + lf))
                r = (int32_t)(__ldg(D.leaf_start + lf) + (int64_t)sfx - 1);
            }
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
  int64_t dir2;            // rank2 / planes / sliced: deep-row base of the block
};

__device__ __forceinline__ void vbs_block_meta(const VbsLookupDesc& d, int64_t blk,
                                               VbsBlockMeta& mt) {
#pragma unroll
  for (int j = 2; j <= kMaxLevels; ++j) mt.m[j - 1] = j <= d.K ? __ldg(d.exist[j - 1] + blk) : 0u;
  mt.dir2 = (d.mode != BSB_DEEP_PACKED && d.K >= 2) ? __ldg(d.dir[1] + blk) : 0;
}

// right-aligned code and length of row lr of block blk, given its BS_1 byte
__device__ __forceinline__ uint64_t vbs_row_code_f(const VbsLookupDesc& d, int64_t blk, int lr,
                                                   const VbsBlockMeta& mt, uint32_t first,
                                                   int& len) {
  const uint32_t below = (1u << lr) - 1u;
  uint64_t code = first;
  len = 1;
  const int64_t q = mt.dir2 + __popc(mt.m[1] & below);
  for (int j = 2; j <= d.K; ++j) {
    const uint32_t w = mt.m[j - 1];
    if (!((w >> lr) & 1u)) break;
    uint32_t byte;
    if (d.mode == BSB_DEEP_SLICED) {
      byte = __ldg(d.deep[j - 1] + ((q & ~int64_t(31)) + swz((int)(q & 31))));
    } else if (d.mode == BSB_DEEP_PLANES) {
      const uint16_t v = __ldg(reinterpret_cast<const uint16_t*>(d.deep[((j - 2) >> 1) + 1]) + q);
      byte = ((j - 2) & 1) ? (v & 0xFFu) : (v >> 8);
    } else if (d.mode == BSB_DEEP_RANK2) {
      byte = __ldg(d.deep[j - 1] + q);
    } else {
      byte = __ldg(d.deep[j - 1] + (__ldg(d.dir[j - 1] + blk) + __popc(w & below)));
    }
    code = (code << 8) | byte;
    len = j;
  }
  return code;
}

__device__ __forceinline__ uint64_t vbs_row_code(const VbsLookupDesc& d, int64_t blk, int lr,
                                                 const VbsBlockMeta& mt, int& len) {
  return vbs_row_code_f(d, blk, lr, mt, __ldg(d.bs1 + (blk * 32 + swz(lr))), len);
}

__device__ __forceinline__ void emit(uint64_t* oc, int64_t* ov, int32_t* ov32, int64_t pos,
                                     uint64_t code_out, int64_t v) {
  if (oc) oc[pos] = code_out;
  if (ov) ov[pos] = v;
  if (ov32) ov32[pos] = (int32_t)v;
}

// Fused bitvector -> values.  Warp per tile of 1024 rows.  Lane = block:
// every block with a selected row has its sectors fetched with 256-bit loads
// (ByteSlice: the K plane sectors; PP-VBS: the BS_1 sector, the existence
// words and the level-2 directory entry) into the warp's shared-memory
// stage, all in flight together; the tile's set rows are compacted into a
// row list; then lane k assembles listed rows k, k+32, ... from the stage
// (PP-VBS deep bytes from HBM), decodes and writes them contiguously.  A bad
// code sets *err (UINT64_MAX when err is the output count).
constexpr int kBitsThreads = 128;

__host__ __device__ constexpr int bits_stage_bytes(bool vbs, int K) {
  return 2048 + (vbs ? 1024 + 128 * (K > 1 ? K - 1 : 0) + 256 : 1024 * K);
}

template <bool VBS, int DK>
__global__ void __launch_bounds__(kBitsThreads) lookup_bits_kernel(
    const uint8_t* __restrict__ slices, int64_t stride, int K, int width,  // ByteSlice
    const __grid_constant__ VbsLookupDesc vd,                              // PP-VBS
    const uint32_t* __restrict__ words, int64_t nb, int64_t ntiles,
    const int64_t* __restrict__ tile_incl, const __grid_constant__ Decoder D,
    uint64_t* __restrict__ oc, int64_t* __restrict__ ov, int32_t* __restrict__ ov32,
    unsigned long long* __restrict__ err) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int KL = VBS ? vd.K : K;
  uint8_t* wbase = dsm + (threadIdx.x >> 5) * bits_stage_bytes(VBS, KL);
  uint16_t* idx = reinterpret_cast<uint16_t*>(wbase);
  uint8_t* stage = wbase + 2048;
  uint32_t* smeta = reinterpret_cast<uint32_t*>(stage + 1024);          // VBS only
  int64_t* sdir = reinterpret_cast<int64_t*>(smeta + 32 * (KL > 1 ? KL - 1 : 0));
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int shift = VBS ? 0 : 8 * K - width;
  bool bad = false;
  int64_t t = warp;
  uint32_t w = 0;
  if (t < ntiles) w = (t * 32 + lane) < nb ? __ldg(words + t * 32 + lane) : 0u;
  for (; t < ntiles; t += nwarps) {
    const int64_t tn = t + nwarps;
    const uint32_t wn = (tn < ntiles && tn * 32 + lane < nb) ? __ldg(words + tn * 32 + lane) : 0u;
    const uint32_t c = __popc(w);
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (total) {
      const int64_t blk = t * 32 + lane;
      if (w) {
        if (VBS) {
          uint32_t v[8];
          ldg256(vd.bs1 + blk * 32, v);
          uint4* dst = reinterpret_cast<uint4*>(stage + lane * 32);
          dst[0] = make_uint4(v[0], v[1], v[2], v[3]);
          dst[1] = make_uint4(v[4], v[5], v[6], v[7]);
          for (int j = 2; j <= KL; ++j) smeta[(j - 2) * 32 + lane] = __ldg(vd.exist[j - 1] + blk);
          sdir[lane] = (vd.mode != BSB_DEEP_PACKED && KL >= 2) ? __ldg(vd.dir[1] + blk) : 0;
        } else {
          for (int j = 0; j < K; ++j) {
            uint32_t v[8];
            ldg256(slices + j * stride + blk * 32, v);
            uint4* dst = reinterpret_cast<uint4*>(stage + j * 1024 + lane * 32);
            dst[0] = make_uint4(v[0], v[1], v[2], v[3]);
            dst[1] = make_uint4(v[4], v[5], v[6], v[7]);
          }
        }
      }
      const uint32_t excl = incl - c;
      const int64_t tbase = t ? __ldg(tile_incl + t - 1) : 0;
      // each lane lists its own block's set rows (ascending)
      uint32_t rest = w;
      uint32_t o = excl;
      while (rest) {
        const int bit = __ffs(rest) - 1;
        rest &= rest - 1;
        idx[o++] = (uint16_t)((lane << 5) | bit);
      }
      __syncwarp();
      for (uint32_t k0 = lane; k0 < total; k0 += 64) {
        uint64_t code[2], pad[2];
        int len[2];
        bool on[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t k = k0 + 32 * u;
          on[u] = k < total;
          const uint32_t r = on[u] ? idx[k] : 0u;
          const int bl = (int)(r >> 5);
          const int lr = (int)(r & 31);
          const int off = bl * 32 + swz(lr);
          if (VBS) {
            VbsBlockMeta mt;
#pragma unroll
            for (int j = 2; j <= kMaxLevels; ++j)
              mt.m[j - 1] = (j <= KL && on[u]) ? smeta[(j - 2) * 32 + bl] : 0u;
            mt.dir2 = sdir[bl];
            code[u] = vbs_row_code_f(vd, t * 32 + bl, lr, mt, stage[off], len[u]);
            pad[u] = code[u] << (8 * (KL - len[u]));
          } else {
            uint64_t cd = 0;
#pragma unroll
            for (int j = 0; j < kMaxLevels; ++j)
              if (j < K) cd = (cd << 8) | stage[j * 1024 + off];
            code[u] = pad[u] = cd >> shift;
            len[u] = 0;
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (!on[u]) continue;
          const int64_t v = decode_value<DK>(D, code[u], pad[u], len[u], bad);
          emit(oc, ov, ov32, tbase + k0 + 32 * u, pad[u], v);
        }
      }
      __syncwarp();
    }
    w = wn;
  }
  if (bad) *err = ~0ull;
}

// Row-id lookup + general decode; kIdsPerThread ids per thread in flight.
__global__ void vbs_lookup_rows_dec_kernel(const __grid_constant__ VbsLookupDesc vd,
                                           const int64_t* __restrict__ rows, int64_t n_ids,
                                           const __grid_constant__ Decoder D,
                                           uint64_t* __restrict__ oc, int64_t* __restrict__ ov,
                                           int32_t* __restrict__ ov32,
                                           unsigned int* __restrict__ err) {
  bool bad = false;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n_ids;
       i0 += nthr * kIdsPerThread) {
    uint64_t code[kIdsPerThread];
    int len[kIdsPerThread];
#pragma unroll
    for (int u = 0; u < kIdsPerThread; ++u) {
      const int64_t i = i0 + u * nthr;
      const int64_t r = i < n_ids ? __ldg(rows + i) : 0;
      const int64_t blk = r >> 5;
      VbsBlockMeta mt;
      vbs_block_meta(vd, blk, mt);
      code[u] = vbs_row_code(vd, blk, (int)(r & 31), mt, len[u]);
    }
#pragma unroll
    for (int u = 0; u < kIdsPerThread; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i >= n_ids) break;
      const uint64_t padded = code[u] << (8 * (vd.K - len[u]));
      const int64_t v = decode_value(D, code[u], padded, len[u], bad);
      emit(oc, ov, ov32, i, padded, v);
    }
  }
  if (bad) atomicOr(err, 1u);
}

static void fill_lookup_desc(VbsLookupDesc& d, const bsb_vbs* col) {
  std::memset(&d, 0, sizeof(d));
  d.bs1 = col->bs1;
  d.K = col->max_len;
  d.mode = col->deep_mode;
  for (int j = 0; j < kMaxLevels; ++j) {
    d.deep[j] = col->deep[j];
    d.exist[j] = col->exist[j];
    d.dir[j] = col->block_dir[j];
  }
}

static int finish_err(unsigned int* err, cudaStream_t s, bool need) {
  if (!need) {
    BSB_CUDA(cudaFreeAsync(err, s));
    return BSB_OK;
  }
  unsigned int h = 0;
  BSB_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(err, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (h) {
    set_error_msg("padded code not in dictionary");
    return BSB_ENOTFOUND;
  }
  return BSB_OK;
}

template <bool VBS>
static int lookup_bits_impl(const bsb_byteslice* bcol, const bsb_vbs* vcol,
                            const uint32_t* words, const bsb_decode* dec, uint64_t* oc,
                            int64_t* ov, int32_t* ov32, uint64_t* n_out_dev, cudaStream_t s) {
  const int64_t n = VBS ? vcol->n_rows : bcol->n_rows;
  const int64_t nb = (n + 31) / 32;
  const int64_t ntiles = (nb + 31) / 32;
  int64_t* tc = nullptr;
  BSB_CUDA(cudaMallocAsync(&tc, (ntiles * 2 + 4) * sizeof(int64_t), s));
  int64_t* incl = tc + ntiles + 1;
  unsigned long long* errw = reinterpret_cast<unsigned long long*>(incl + ntiles + 1);
  const int grid = grid_for_l(ntiles * 32, 256);
  tile_popc_kernel<<<grid, 256, 0, s>>>(words, nb, ntiles, tc);
  BSB_LAUNCH_CHECK();
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, tc, incl, ntiles, s);
  void* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, tb + 16, s));
  cub::DeviceScan::InclusiveSum(tmp, tb, tc, incl, ntiles, s);
  BSB_LAUNCH_CHECK();
  if (n_out_dev)
    BSB_CUDA(cudaMemcpyAsync(n_out_dev, incl + ntiles - 1, 8, cudaMemcpyDeviceToDevice, s));
  else
    BSB_CUDA(cudaMemsetAsync(errw, 0, 8, s));
  Decoder D;
  fill_decoder(D, dec);
  VbsLookupDesc vd;
  std::memset(&vd, 0, sizeof(vd));
  if (VBS) fill_lookup_desc(vd, vcol);
  const int wpb = kBitsThreads / 32;
  const int smem = wpb * bits_stage_bytes(VBS, VBS ? vcol->max_len : bcol->n_slices);
  auto launch = [&](auto kern) -> int {
    int per_sm = 0;
    BSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBitsThreads, smem));
    const int bgrid = (int)std::min<int64_t>((ntiles + wpb - 1) / wpb,
                                             (int64_t)sm_count() * (per_sm < 1 ? 1 : per_sm));
    kern<<<bgrid < 1 ? 1 : bgrid, kBitsThreads, smem, s>>>(
        VBS ? nullptr : bcol->slices, VBS ? 0 : bcol->stride, VBS ? 0 : bcol->n_slices,
        VBS ? 0 : bcol->width_bits, vd, words, nb, ntiles, incl, D, oc, ov, ov32,
        n_out_dev ? reinterpret_cast<unsigned long long*>(n_out_dev) : errw);
    BSB_LAUNCH_CHECK();
    return BSB_OK;
  };
  int rc;
  switch (D.kind) {
    case 0: rc = launch(lookup_bits_kernel<VBS, 0>); break;
    case 1: rc = launch(lookup_bits_kernel<VBS, 1>); break;
    case 2: rc = launch(lookup_bits_kernel<VBS, 2>); break;
    default: rc = launch(lookup_bits_kernel<VBS, 3>); break;
  }
  if (rc != BSB_OK) return rc;
  BSB_CUDA(cudaFreeAsync(tmp, s));
  if (n_out_dev || D.kind == 0) {
    BSB_CUDA(cudaFreeAsync(tc, s));
    return BSB_OK;
  }
  unsigned long long h = 0;
  BSB_CUDA(cudaMemcpyAsync(&h, errw, 8, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(tc, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (h) {
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

extern "C" int bsb_vbs_lookup_rows_dec(const bsb_vbs* col, const int64_t* rows, int64_t n_ids,
                                       const bsb_decode* dec, uint64_t* out_padded,
                                       int64_t* out_values, int32_t* out_values32,
                                       uint32_t* err_dev, void* stream) {
  if (!col || n_ids < 0 || (n_ids > 0 && !rows)) return BSB_EINVAL;
  if (dec && (dec->kind == 1 || dec->kind > 3)) return BSB_EINVAL;
  if (n_ids == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  Decoder D;
  fill_decoder(D, dec);
  VbsLookupDesc vd;
  fill_lookup_desc(vd, col);
  unsigned int* err = err_dev;
  if (!err) {
    BSB_CUDA(cudaMallocAsync(&err, 4, s));
    BSB_CUDA(cudaMemsetAsync(err, 0, 4, s));
  }
  vbs_lookup_rows_dec_kernel<<<grid_for_l((n_ids + kIdsPerThread - 1) / kIdsPerThread, 256), 256,
                               0, s>>>(vd, rows, n_ids, D, out_padded, out_values, out_values32,
                                       err);
  BSB_LAUNCH_CHECK();
  if (err_dev) return BSB_OK;
  return finish_err(err, s, D.kind >= 2);
}
