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

// lookup_byteslice (byteslice.py:143-158) + decode_ranks (dictionary.py:413-414)
__global__ void bs_lookup_kernel(const uint8_t* __restrict__ slices, int64_t stride, int K,
                                 int width, const int64_t* __restrict__ rows, int64_t n_ids,
                                 uint64_t* __restrict__ out_codes,
                                 const int64_t* __restrict__ rank_values,
                                 int64_t* __restrict__ out_values,
                                 int32_t* __restrict__ out_values32) {
  const int shift = 8 * K - width;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_ids;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = __ldg(rows + i);
    const int64_t pos = (r & ~int64_t(31)) + swz((int)(r & 31));
    uint64_t c = 0;
#pragma unroll 4
    for (int j = 0; j < K; ++j) c = (c << 8) | __ldg(slices + (int64_t)j * stride + pos);
    c >>= shift;
    if (out_codes) out_codes[i] = c;
    if (rank_values) {
      const int64_t v = __ldg(rank_values + c);
      if (out_values) out_values[i] = v;
      if (out_values32) out_values32[i] = (int32_t)v;
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
  bs_lookup_kernel<<<grid_for_l(n_ids, 256), 256, 0, s>>>(
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
