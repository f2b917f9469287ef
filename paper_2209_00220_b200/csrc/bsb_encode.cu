// bsb_encode.cu -- column encoders: frequency table + ranks (device radix
// sort), encode_rows, PPE numerical code assignment (host, O(distinct)),
// per-row code gather and the Zipf inverse-CDF sampler.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "bsb_common.cuh"

namespace bsb {

static int grid_e(int64_t items, int threads, int cap = 148 * 16) {
  int64_t g = (items + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

template <typename KeyT, typename IdxT>
__global__ void make_keys_kernel(const int64_t* __restrict__ v, int64_t n, int64_t vmin,
                                 KeyT* __restrict__ keys, IdxT* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (KeyT)((uint64_t)v[i] - (uint64_t)vmin);
    idx[i] = (IdxT)i;
  }
}

template <typename KeyT>
__global__ void head_flags_kernel(const KeyT* __restrict__ k, int64_t n, int64_t* __restrict__ f) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    f[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

template <typename KeyT, typename IdxT>
__global__ void emit_ranks_kernel(const KeyT* __restrict__ k, const IdxT* __restrict__ idx,
                                  const int64_t* __restrict__ incl, int64_t n, int64_t vmin,
                                  int64_t* __restrict__ ranks, int64_t* __restrict__ uniq,
                                  int64_t* __restrict__ start) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = incl[i] - 1;
    if (ranks) ranks[idx[i]] = r;
    if (i == 0 || k[i] != k[i - 1]) {
      uniq[r] = (int64_t)((uint64_t)k[i] + (uint64_t)vmin);
      start[r] = i;
    }
  }
}

__global__ void counts_kernel(const int64_t* __restrict__ start, int64_t D, int64_t n,
                              int64_t* __restrict__ counts) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < D;
       r += (int64_t)gridDim.x * blockDim.x)
    counts[r] = (r + 1 < D ? start[r + 1] : n) - start[r];
}

template <typename KeyT, typename IdxT>
static int freq_impl(const int64_t* values, int64_t n, int64_t vmin, int end_bit,
                     int64_t* uniq, int64_t* counts, int64_t* ranks, int64_t* D_host,
                     cudaStream_t s) {
  KeyT *k0 = nullptr, *k1 = nullptr;
  IdxT *i0 = nullptr, *i1 = nullptr;
  int64_t* flags = nullptr;
  BSB_CUDA(cudaMallocAsync(&k0, n * sizeof(KeyT), s));
  BSB_CUDA(cudaMallocAsync(&k1, n * sizeof(KeyT), s));
  BSB_CUDA(cudaMallocAsync(&i0, n * sizeof(IdxT), s));
  BSB_CUDA(cudaMallocAsync(&i1, n * sizeof(IdxT), s));
  BSB_CUDA(cudaMallocAsync(&flags, n * sizeof(int64_t), s));
  make_keys_kernel<KeyT, IdxT><<<grid_e(n, 256), 256, 0, s>>>(values, n, vmin, k0, i0);
  BSB_LAUNCH_CHECK();
  cub::DoubleBuffer<KeyT> kb(k0, k1);
  cub::DoubleBuffer<IdxT> ib(i0, i1);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, ib, (int64_t)n, 0, end_bit, s);
  void* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, ib, (int64_t)n, 0, end_bit, s);
  BSB_LAUNCH_CHECK();
  BSB_CUDA(cudaFreeAsync(tmp, s));
  const KeyT* ks = kb.Current();
  const IdxT* is = ib.Current();
  head_flags_kernel<KeyT><<<grid_e(n, 256), 256, 0, s>>>(ks, n, flags);
  BSB_LAUNCH_CHECK();
  tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, flags, flags, n, s);
  BSB_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, flags, flags, n, s);
  BSB_LAUNCH_CHECK();
  BSB_CUDA(cudaFreeAsync(tmp, s));
  // start offsets of each run reuse the alternate key buffer when it fits
  int64_t* start = nullptr;
  BSB_CUDA(cudaMallocAsync(&start, n * sizeof(int64_t), s));
  emit_ranks_kernel<KeyT, IdxT><<<grid_e(n, 256), 256, 0, s>>>(ks, is, flags, n, vmin, ranks,
                                                               uniq, start);
  BSB_LAUNCH_CHECK();
  int64_t D = 0;
  BSB_CUDA(cudaMemcpyAsync(&D, flags + (n - 1), 8, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  counts_kernel<<<grid_e(D, 256), 256, 0, s>>>(start, D, n, counts);
  BSB_LAUNCH_CHECK();
  BSB_CUDA(cudaFreeAsync(start, s));
  BSB_CUDA(cudaFreeAsync(flags, s));
  BSB_CUDA(cudaFreeAsync(k0, s));
  BSB_CUDA(cudaFreeAsync(k1, s));
  BSB_CUDA(cudaFreeAsync(i0, s));
  BSB_CUDA(cudaFreeAsync(i1, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  *D_host = D;
  return BSB_OK;
}

__global__ void encode_rows_kernel(const int64_t* __restrict__ v, int64_t n,
                                   const int64_t* __restrict__ table, int64_t D,
                                   int64_t* __restrict__ ranks, unsigned int* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = v[i];
    int64_t lo = 0, hi = D;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(table + mid) < x)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo >= D || __ldg(table + lo) != x) {
      atomicOr(err, 1u);
      lo = 0;
    }
    ranks[i] = lo;
  }
}

__global__ void gather_codes_kernel(const int64_t* __restrict__ ranks, int64_t n,
                                    const uint64_t* __restrict__ codes,
                                    const uint8_t* __restrict__ lens,
                                    uint64_t* __restrict__ codes_out,
                                    uint8_t* __restrict__ lens_out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = ranks[i];
    if (codes_out) codes_out[i] = __ldg(codes + r);
    if (lens_out) lens_out[i] = __ldg(lens + r);
  }
}

// searchsorted(cdf, u, side="right") (datagen.py:56)
__global__ void zipf_kernel(const double* __restrict__ u, int64_t n,
                            const double* __restrict__ cdf, int64_t domain,
                            int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = u[i];
    int64_t lo = 0, hi = domain;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(cdf + mid) <= x)
        lo = mid + 1;
      else
        hi = mid;
    }
    out[i] = lo;
  }
}

}  // namespace bsb

using namespace bsb;

extern "C" int bsb_freq_table(const int64_t* values, int64_t n, int64_t* uniq_out,
                              int64_t* counts_out, int64_t* ranks_out, int64_t* n_distinct_host,
                              void* stream) {
  if (!values || n <= 0 || !uniq_out || !counts_out || !n_distinct_host) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  int64_t* mm = nullptr;
  BSB_CUDA(cudaMallocAsync(&mm, 16, s));
  size_t tb = 0, tb2 = 0;
  cub::DeviceReduce::Min(nullptr, tb, values, mm, n, s);
  cub::DeviceReduce::Max(nullptr, tb2, values, mm + 1, n, s);
  void* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, std::max(tb, tb2) + 16, s));
  cub::DeviceReduce::Min(tmp, tb, values, mm, n, s);
  cub::DeviceReduce::Max(tmp, tb2, values, mm + 1, n, s);
  BSB_LAUNCH_CHECK();
  int64_t h[2];
  BSB_CUDA(cudaMemcpyAsync(h, mm, 16, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(tmp, s));
  BSB_CUDA(cudaFreeAsync(mm, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  const uint64_t range = (uint64_t)h[1] - (uint64_t)h[0];
  int bits = 0;
  while (bits < 64 && (range >> bits) != 0) ++bits;
  if (bits == 0) bits = 1;
  const bool small_idx = n < (int64_t(1) << 31);
  if (bits <= 32) {
    if (small_idx)
      return freq_impl<uint32_t, int32_t>(values, n, h[0], bits, uniq_out, counts_out, ranks_out,
                                          n_distinct_host, s);
    return freq_impl<uint32_t, int64_t>(values, n, h[0], bits, uniq_out, counts_out, ranks_out,
                                        n_distinct_host, s);
  }
  if (small_idx)
    return freq_impl<uint64_t, int32_t>(values, n, h[0], bits, uniq_out, counts_out, ranks_out,
                                        n_distinct_host, s);
  return freq_impl<uint64_t, int64_t>(values, n, h[0], bits, uniq_out, counts_out, ranks_out,
                                      n_distinct_host, s);
}

extern "C" int bsb_encode_rows(const int64_t* values, int64_t n, const int64_t* table_values,
                               int64_t n_dict, int64_t* ranks_out, void* stream) {
  if (!values || n < 0 || !table_values || n_dict <= 0 || !ranks_out) return BSB_EINVAL;
  if (n == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  unsigned int* err = nullptr;
  BSB_CUDA(cudaMallocAsync(&err, 4, s));
  BSB_CUDA(cudaMemsetAsync(err, 0, 4, s));
  encode_rows_kernel<<<grid_e(n, 256), 256, 0, s>>>(values, n, table_values, n_dict, ranks_out,
                                                    err);
  BSB_LAUNCH_CHECK();
  unsigned int h = 0;
  BSB_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(err, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (h) {
    set_error_msg("value missing from dictionary");
    return BSB_EKEY;
  }
  return BSB_OK;
}

extern "C" int bsb_gather_codes(const int64_t* ranks, int64_t n, const uint64_t* dict_codes,
                                const uint8_t* dict_lens, uint64_t* codes_out, uint8_t* lens_out,
                                void* stream) {
  if (!ranks || n < 0 || !dict_codes || !dict_lens) return BSB_EINVAL;
  if (n == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  gather_codes_kernel<<<grid_e(n, 256), 256, 0, s>>>(ranks, n, dict_codes, dict_lens, codes_out,
                                                     lens_out);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

extern "C" int bsb_zipf_from_uniform(const double* u, int64_t n, const double* cdf,
                                     int64_t domain, int64_t* values_out, void* stream) {
  if (!u || n < 0 || !cdf || domain <= 0 || !values_out) return BSB_EINVAL;
  if (n == 0) return BSB_OK;
  cudaStream_t s = as_stream(stream);
  zipf_kernel<<<grid_e(n, 256), 256, 0, s>>>(u, n, cdf, domain, values_out);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

// ------------------------------------------------------------------------
// ppe_numerical (dictionary.py:148-196), host side: O(D log 255) per level.
namespace {

int suffix_bytes(int64_t m) {  // least beta with 256^beta >= m (0 for m <= 1)
  int beta = 0;
  while (beta < 8 && (uint64_t(1) << (8 * beta)) < (uint64_t)m) ++beta;
  return beta;
}

struct Node {
  int64_t s, e;
  int depth;
  uint64_t prefix;
};

}  // namespace

extern "C" int bsb_ppe_numerical_host(const int64_t* w, int64_t n, uint64_t* codes,
                                      uint8_t* lens) {
  if (!w || n <= 0 || !codes || !lens) return BSB_EINVAL;
  for (int64_t i = 0; i < n; ++i)
    if (w[i] < 0) {
      set_error_msg("negative weight");
      return BSB_EINVAL;
    }
  std::vector<Node> todo;
  todo.push_back({0, n, 0, 0});
  std::vector<int64_t> idx;
  while (!todo.empty()) {
    const Node nd = todo.back();
    todo.pop_back();
    const int64_t size = nd.e - nd.s;
    if (size == 0) continue;
    if (size < 256 || nd.depth >= 2) {
      const int beta = suffix_bytes(size + 1);
      for (int64_t i = 0; i < size; ++i) {
        codes[nd.s + i] = (beta >= 8 ? 0 : (nd.prefix << (8 * beta))) + (uint64_t)(i + 1);
        lens[nd.s + i] = (uint8_t)(nd.depth + beta);
      }
      continue;
    }
    // 255 heaviest values (ties -> lower index) become slots 1..255 in value order
    idx.resize(size);
    std::iota(idx.begin(), idx.end(), nd.s);
    std::partial_sort(idx.begin(), idx.begin() + 255, idx.end(), [&](int64_t a, int64_t b) {
      return w[a] != w[b] ? w[a] > w[b] : a < b;
    });
    std::vector<int64_t> slots(idx.begin(), idx.begin() + 255);
    std::sort(slots.begin(), slots.end());
    for (int t = 0; t < 255; ++t) {
      codes[slots[t]] = (nd.prefix << 8) + (uint64_t)(t + 1);
      lens[slots[t]] = (uint8_t)(nd.depth + 1);
    }
    int64_t prev = nd.s - 1;
    for (int t = 0; t < 256; ++t) {
      const int64_t cs = prev + 1;
      const int64_t ce = t < 255 ? slots[t] : nd.e;
      if (ce > cs) todo.push_back({cs, ce, nd.depth + 1, (nd.prefix << 8) | (uint64_t)t});
      if (t < 255) prev = slots[t];
    }
  }
  return BSB_OK;
}
