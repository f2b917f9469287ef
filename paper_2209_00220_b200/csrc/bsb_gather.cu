// bsb_gather.cu -- locality for row-id gathers.
//
// A lookup of a row-id list in random order (cfg3's unsorted ids) touches one
// random 32-byte sector per slice per id.  Sorting the ids first turns the
// gather into a forward walk over the column (ids that share a block share
// its sectors, and DRAM pages are visited in order); the looked-up values are
// then scattered back to input order.  The host wrappers
// (lookup_*_rows(order="auto")) use this for large unsorted lists.
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
