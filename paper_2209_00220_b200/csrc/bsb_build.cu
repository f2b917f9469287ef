// bsb_build.cu -- device layout construction (ByteSlice + PP-VBS) and the
// misc C-ABI entry points (version, errors, stride).
#include <cub/device/device_scan.cuh>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "bsb_common.cuh"

namespace bsb {

static thread_local std::string g_last_error;

void set_error(const char* where, cudaError_t err) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%s: %s (%s)", where, cudaGetErrorString(err),
                cudaGetErrorName(err));
  g_last_error = buf;
}
void set_error_msg(const char* msg) { g_last_error = msg; }

void ensure_init() {
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

static int g_ctas_cap = -1;
int ctas_per_sm_cap() {
  if (g_ctas_cap < 0) {
    const char* e = std::getenv("BSB_CTAS_PER_SM");
    g_ctas_cap = e ? std::atoi(e) : 0;
  }
  return g_ctas_cap;
}
void set_ctas_per_sm_cap(int v) { g_ctas_cap = v < 0 ? 0 : v; }

int sm_count() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
  }
  return cached;
}

static int grid_for(int64_t items, int threads, int cap = 148 * 16) {
  int64_t g = (items + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// ------------------------------------------------------------- ByteSlice

// Warp per 32-row block: lane r validates and aligns row r's code
// (byteslice.py:52-73), then every plane's block is written in the
// bit-plane layout (bsb_common.cuh, "BP32") with 8 ballots.
template <typename CodeT>
__global__ void bs_build_kernel(const CodeT* __restrict__ codes, int64_t n, int width, int K,
                                uint8_t* __restrict__ slices, int64_t stride,
                                unsigned int* __restrict__ err) {
  const int shift = 8 * K - width;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < stride / 32; b += nwarps) {
    const int64_t r = b * 32 + lane;
    uint64_t c = 0;
    if (r < n) {
      const CodeT v = codes[r];
      if (v < 0) {
        atomicOr(err, 1u);
      } else {
        c = (uint64_t)v;
        if (width < 64 && (c >> width) != 0) atomicOr(err, 1u);
      }
    }
    const uint64_t a = shift >= 64 ? 0 : (c << shift);
    for (int j = 0; j < K; ++j)
      bp_store_block(slices + (int64_t)j * stride + b * 32,
                     (uint32_t)(a >> (8 * (K - 1 - j))) & 0xFFu, lane);
  }
}

// Reference planes (row order, byteslice.py:68): out[j][r]
__global__ void bs_export_kernel(const uint8_t* __restrict__ slices, int64_t stride, int K,
                                 int64_t npad, uint8_t* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < npad;
       r += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < K; ++j) {
      uint32_t w[8];
      ldg256(slices + (int64_t)j * stride + (r >> 5) * 32, w);
      out[(int64_t)j * npad + r] = (uint8_t)bp_byte(w, (int)(r & 31));
    }
  }
}

template <typename CodeT>
static int bs_build_impl(const CodeT* codes, int64_t n, int32_t width, uint8_t* slices,
                         int64_t stride, cudaStream_t s) {
  if (!codes || !slices || n <= 0) return BSB_EINVAL;
  if (width < 1 || width > 64) return BSB_ERANGE;
  if (stride < n || (stride % kTileRows) != 0) return BSB_EINVAL;
  const int K = (width + 7) / 8;
  unsigned int* err = nullptr;
  BSB_CUDA(cudaMallocAsync(&err, sizeof(unsigned int), s));
  BSB_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned int), s));
  bs_build_kernel<CodeT><<<grid_for(stride, 256), 256, 0, s>>>(codes, n, width, K, slices,
                                                               stride, err);  // warp per block
  BSB_LAUNCH_CHECK();
  unsigned int h = 0;
  BSB_CUDA(cudaMemcpyAsync(&h, err, sizeof(h), cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(err, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (h) {
    set_error_msg("code wider than declared width");
    return BSB_ERANGE;
  }
  return BSB_OK;
}

// ---------------------------------------------------------------- PP-VBS

__global__ void vbs_plan_kernel(const uint64_t* __restrict__ codes,
                                const uint8_t* __restrict__ lens, int64_t n,
                                unsigned long long* __restrict__ level_rows,
                                unsigned int* __restrict__ maxlen, unsigned int* __restrict__ err) {
  unsigned long long loc[kMaxLevels];
#pragma unroll
  for (int j = 0; j < kMaxLevels; ++j) loc[j] = 0;
  unsigned int mx = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned l = lens[r];
    if (l < 1 || l > 8) {
      atomicOr(err, 1u);
      continue;
    }
    if (l < 8 && (codes[r] >> (8 * l)) != 0) atomicOr(err, 2u);
    mx = l > mx ? l : mx;
#pragma unroll
    for (int j = 0; j < kMaxLevels; ++j) loc[j] += (l > (unsigned)j);
  }
#pragma unroll
  for (int j = 0; j < kMaxLevels; ++j) {
    unsigned long long v = loc[j];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(level_rows + j, v);
  }
  mx = __reduce_max_sync(kFull, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(maxlen, mx);
}

// One warp per block of 32 rows: first-byte plane, existence words, counts.
__global__ void vbs_exist_kernel(const uint64_t* __restrict__ codes,
                                 const uint8_t* __restrict__ lens, int64_t n, int64_t nbpad,
                                 int K, uint8_t* __restrict__ bs1, uint32_t* const* exist,
                                 int64_t* __restrict__ counts /* (K-1) x nbpad */) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = warp; b < nbpad; b += nwarps) {
    const int64_t r = b * 32 + lane;
    unsigned l = 0;
    uint64_t c = 0;
    if (r < n) {
      l = lens[r];
      c = codes[r];
    }
    bp_store_block(bs1 + b * 32, l ? (uint32_t)(c >> (8 * (l - 1))) & 0xFFu : 0u, lane);
    for (int j = 2; j <= K; ++j) {
      const uint32_t bal = __ballot_sync(kFull, l >= (unsigned)j);
      if (lane == 0) {
        exist[j - 1][b] = bal;
        counts[(int64_t)(j - 2) * nbpad + b] = __popc(bal);
      }
    }
  }
}

// Deep rows in row order: SLICED gathers each deep row's (code, length) at
// its deep-row index q (the rank of the row among rows with >= 2 bytes, from
// the level-2 directory); PACKED writes the reference packing (vbs.py:98-100).
__global__ void vbs_scatter_kernel(const uint64_t* __restrict__ codes,
                                   const uint8_t* __restrict__ lens, int64_t n, int K, int mode,
                                   uint8_t* const* deep, const uint32_t* const* exist,
                                   const int64_t* const* dir, uint64_t* __restrict__ dcode,
                                   uint8_t* __restrict__ dlen) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned l = lens[r];
    if (l < 2) continue;
    const uint64_t c = codes[r];
    const int64_t b = r >> 5;
    const uint32_t below = (1u << (r & 31)) - 1u;
    if (mode == BSB_DEEP_SLICED) {
      const int64_t q = dir[1][b] + __popc(exist[1][b] & below);
      dcode[q] = c;
      dlen[q] = (uint8_t)l;
    } else {
      for (int j = 2; j <= (int)l; ++j) {
        const uint32_t w = exist[j - 1][b];
        const int64_t pos = dir[j - 1][b] + __popc(w & below);
        deep[j - 1][pos] = (uint8_t)(c >> (8 * (l - j)));
      }
    }
  }
}

// SLICED deep planes, warp per 32-deep-row block: byte j of every deep row
// (0 where the code is shorter) in the bit-plane layout, byte 1 in deep[0]
// when allocated, and rexist[j] = "deep row has byte j+1" (j >= 2).
__global__ void vbs_deep_planes_kernel(const uint64_t* __restrict__ dcode,
                                       const uint8_t* __restrict__ dlen, int64_t cnt2, int K,
                                       uint8_t* const* deep, uint32_t* const* rexist) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ndb = (cnt2 + 31) / 32;
  for (int64_t db = warp; db < ndb; db += nwarps) {
    const int64_t q = db * 32 + lane;
    const unsigned l = q < cnt2 ? dlen[q] : 0u;
    const uint64_t c = q < cnt2 ? dcode[q] : 0ull;
    if (deep[0])
      bp_store_block(deep[0] + db * 32, l ? (uint32_t)(c >> (8 * (l - 1))) & 0xFFu : 0u, lane);
    for (int j = 2; j <= K; ++j) {
      const uint32_t byte = j <= (int)l ? (uint32_t)(c >> (8 * (l - j))) & 0xFFu : 0u;
      bp_store_block(deep[j - 1] + db * 32, byte, lane);
      if (j < K) {
        const uint32_t bal = __ballot_sync(kFull, (int)l >= j + 1);
        if (lane == 0) rexist[j][db] = bal;
      }
    }
  }
}

// Reference-packed bytes of one deep level from either device packing.
__global__ void vbs_export_level_kernel(int64_t n, int level, int mode,
                                        const uint8_t* __restrict__ deep_l,
                                        const uint32_t* __restrict__ exist_l,
                                        const uint32_t* __restrict__ exist_2,
                                        const int64_t* __restrict__ dir_src,
                                        const int64_t* __restrict__ ref_dir,
                                        uint8_t* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = r >> 5;
    const uint32_t below = (1u << (r & 31)) - 1u;
    const uint32_t w = exist_l[b];
    if (!((w >> (r & 31)) & 1u)) continue;
    const int64_t src = mode != BSB_DEEP_PACKED ? dir_src[b] + __popc(exist_2[b] & below)
                                                : dir_src[b] + __popc(w & below);
    uint8_t byte;
    if (mode == BSB_DEEP_SLICED) {
      uint32_t v[8];
      ldg256(deep_l + (src >> 5) * 32, v);
      byte = (uint8_t)bp_byte(v, (int)(src & 31));
    } else {
      byte = deep_l[src];
    }
    out[ref_dir[b] + __popc(w & below)] = byte;
  }
}

__global__ void popc_words_kernel(const uint32_t* __restrict__ w, int64_t nb,
                                  int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __popc(w[i]);
}

__global__ void vbs_export_kernel(const uint8_t* __restrict__ bs1, int64_t npad,
                                  uint8_t* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < npad;
       r += (int64_t)gridDim.x * blockDim.x)
  {
    uint32_t v[8];
    ldg256(bs1 + (r >> 5) * 32, v);
    out[r] = (uint8_t)bp_byte(v, (int)(r & 31));
  }
}

struct PtrTable {
  uint8_t* deep[kMaxLevels];
  uint32_t* exist[kMaxLevels];
  int64_t* dir[kMaxLevels];
  uint32_t* rexist[kMaxLevels];
};

}  // namespace bsb

using namespace bsb;

extern "C" const char* bsb_version(void) { return "bytestore_b200 0.1 sm_100a"; }
extern "C" const char* bsb_last_error(void) { return g_last_error.c_str(); }
extern "C" int64_t bsb_stride_for(int64_t n_rows) {
  if (n_rows <= 0) return kTileRows;
  return ((n_rows + kTileRows - 1) / kTileRows) * kTileRows;
}
extern "C" void bsb_stats_layout(int32_t* w, int32_t* b, int32_t* t, int32_t* s, int32_t* l) {
  if (w) *w = 0;
  if (b) *b = 8;
  if (t) *t = 16;
  if (s) *s = 17;
  if (l) *l = 18;
}

extern "C" int bsb_byteslice_build(const uint64_t* codes, int64_t n_rows, int32_t width_bits,
                                   uint8_t* slices, int64_t stride, void* stream) {
  // uint64 codes: reinterpret as unsigned (no sign check)
  if (!codes || !slices || n_rows <= 0) return BSB_EINVAL;
  if (width_bits < 1 || width_bits > 64) return BSB_ERANGE;
  return bs_build_impl<unsigned long long>(reinterpret_cast<const unsigned long long*>(codes),
                                           n_rows, width_bits, slices, stride,
                                           as_stream(stream));
}

extern "C" int bsb_byteslice_build_ranks(const int64_t* ranks, int64_t n_rows,
                                         int32_t width_bits, uint8_t* slices, int64_t stride,
                                         void* stream) {
  return bs_build_impl<long long>(reinterpret_cast<const long long*>(ranks), n_rows,
                                  width_bits, slices, stride, as_stream(stream));
}

extern "C" int bsb_byteslice_export(const bsb_byteslice* col, uint8_t* out, void* stream) {
  if (!col || !out) return BSB_EINVAL;
  const int64_t npad = (col->n_rows + 31) / 32 * 32;
  cudaStream_t s = as_stream(stream);
  bs_export_kernel<<<grid_for(npad, 256), 256, 0, s>>>(col->slices, col->stride, col->n_slices,
                                                       npad, out);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

extern "C" int bsb_vbs_plan(const uint64_t* codes, const uint8_t* lens, int64_t n_rows,
                            int32_t* max_len_host, int64_t* level_rows_host, void* stream) {
  if (!codes || !lens || n_rows <= 0 || !max_len_host || !level_rows_host) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  struct Scratch {
    unsigned long long rows[kMaxLevels];
    unsigned int maxlen;
    unsigned int err;
  };
  Scratch* d = nullptr;
  BSB_CUDA(cudaMallocAsync(&d, sizeof(Scratch), s));
  BSB_CUDA(cudaMemsetAsync(d, 0, sizeof(Scratch), s));
  vbs_plan_kernel<<<grid_for(n_rows, 256, 148 * 8), 256, 0, s>>>(codes, lens, n_rows, d->rows,
                                                                 &d->maxlen, &d->err);
  BSB_LAUNCH_CHECK();
  Scratch h;
  BSB_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(d, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (h.err & 1u) {
    set_error_msg("code lengths must be 1..8 bytes");
    return BSB_ERANGE;
  }
  if (h.err & 2u) {
    set_error_msg("code wider than its declared length");
    return BSB_ERANGE;
  }
  *max_len_host = (int32_t)h.maxlen;
  for (int j = 0; j < kMaxLevels; ++j) level_rows_host[j] = (int64_t)h.rows[j];
  return BSB_OK;
}

extern "C" int bsb_vbs_build(const uint64_t* codes, const uint8_t* lens, const bsb_vbs* col,
                             void* stream) {
  if (!codes || !lens || !col || col->n_rows <= 0) return BSB_EINVAL;
  const int K = col->max_len;
  if (K < 1 || K > kMaxLevels) return BSB_ERANGE;
  if (col->stride < col->n_rows || col->stride % kTileRows) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int64_t n = col->n_rows;
  const int64_t nbpad = col->stride / 32;
  PtrTable h;
  std::memset(&h, 0, sizeof(h));
  const int mode = col->deep_mode;
  if (mode != BSB_DEEP_PACKED && mode != BSB_DEEP_SLICED) return BSB_EINVAL;
  if (mode == BSB_DEEP_SLICED) h.deep[0] = const_cast<uint8_t*>(col->deep[0]);  // optional
  for (int j = 1; j < K; ++j) {
    const bool need_dir = mode == BSB_DEEP_PACKED || j == 1;
    const bool need_rex = mode == BSB_DEEP_SLICED && j >= 2;
    if (!col->deep[j] || !col->exist[j] || (need_dir && !col->block_dir[j]) ||
        (need_rex && !col->rexist[j]))
      return BSB_EINVAL;
    h.deep[j] = const_cast<uint8_t*>(col->deep[j]);
    h.exist[j] = const_cast<uint32_t*>(col->exist[j]);
    h.dir[j] = const_cast<int64_t*>(col->block_dir[j]);
    h.rexist[j] = const_cast<uint32_t*>(col->rexist[j]);
  }
  PtrTable* dt = nullptr;
  int64_t* counts = nullptr;
  BSB_CUDA(cudaMallocAsync(&dt, sizeof(PtrTable), s));
  BSB_CUDA(cudaMemcpyAsync(dt, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  const int64_t ncnt = (int64_t)(K > 1 ? K - 1 : 1) * nbpad;
  BSB_CUDA(cudaMallocAsync(&counts, ncnt * sizeof(int64_t), s));
  vbs_exist_kernel<<<grid_for(nbpad * 32, 256, 148 * 16), 256, 0, s>>>(
      codes, lens, n, nbpad, K, const_cast<uint8_t*>(col->bs1), dt->exist, counts);
  BSB_LAUNCH_CHECK();
  // block_dir[j] = [0, inclusive prefix of per-block counts]
  for (int j = 1; j < K; ++j) {
    if (mode != BSB_DEEP_PACKED && j > 1) break;  // one shared level-2 directory
    BSB_CUDA(cudaMemsetAsync(h.dir[j], 0, sizeof(int64_t), s));
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, counts + (int64_t)(j - 1) * nbpad,
                                  h.dir[j] + 1, nbpad, s);
    void* tmp = nullptr;
    BSB_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, s));
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, counts + (int64_t)(j - 1) * nbpad,
                                  h.dir[j] + 1, nbpad, s);
    BSB_LAUNCH_CHECK();
    BSB_CUDA(cudaFreeAsync(tmp, s));
  }
  if (K > 1) {
    uint64_t* dcode = nullptr;
    uint8_t* dlen = nullptr;
    int64_t cnt2 = 0;
    if (mode == BSB_DEEP_SLICED) {
      // deep-row count = level-2 directory total
      BSB_CUDA(cudaMemcpyAsync(&cnt2, h.dir[1] + nbpad, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               s));
      BSB_CUDA(cudaStreamSynchronize(s));
      if (cnt2 > 0) {
        BSB_CUDA(cudaMallocAsync(&dcode, (size_t)cnt2 * 8, s));
        BSB_CUDA(cudaMallocAsync(&dlen, (size_t)cnt2, s));
      }
      for (int j = 2; j < K; ++j)
        BSB_CUDA(cudaMemsetAsync(h.rexist[j], 0, (size_t)((cnt2 + 31) / 32) * 4, s));
    }
    vbs_scatter_kernel<<<grid_for(n, 256), 256, 0, s>>>(codes, lens, n, K, mode, dt->deep,
                                                         (const uint32_t* const*)dt->exist,
                                                         (const int64_t* const*)dt->dir, dcode,
                                                         dlen);
    BSB_LAUNCH_CHECK();
    if (mode == BSB_DEEP_SLICED && cnt2 > 0) {
      vbs_deep_planes_kernel<<<grid_for(cnt2, 256), 256, 0, s>>>(dcode, dlen, cnt2, K, dt->deep,
                                                                 dt->rexist);
      BSB_LAUNCH_CHECK();
      BSB_CUDA(cudaFreeAsync(dcode, s));
      BSB_CUDA(cudaFreeAsync(dlen, s));
    }
  }
  BSB_CUDA(cudaFreeAsync(counts, s));
  BSB_CUDA(cudaFreeAsync(dt, s));
  BSB_CUDA(cudaStreamSynchronize(s));  // h/dt lifetime
  return BSB_OK;
}

extern "C" int bsb_vbs_export_bs1(const bsb_vbs* col, uint8_t* out, void* stream) {
  if (!col || !out) return BSB_EINVAL;
  const int64_t npad = (col->n_rows + 31) / 32 * 32;
  cudaStream_t s = as_stream(stream);
  vbs_export_kernel<<<grid_for(npad, 256), 256, 0, s>>>(col->bs1, npad, out);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

extern "C" int bsb_vbs_export_level(const bsb_vbs* col, int32_t level, uint8_t* out_bytes,
                                    int64_t* out_dir, void* stream) {
  if (!col || !out_bytes || !out_dir || level < 2 || level > col->max_len) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int64_t n = col->n_rows;
  const int64_t nb = (n + 31) / 32;
  int64_t* cnt = nullptr;
  BSB_CUDA(cudaMallocAsync(&cnt, nb * sizeof(int64_t), s));
  popc_words_kernel<<<grid_for(nb, 256), 256, 0, s>>>(col->exist[level - 1], nb, cnt);
  BSB_LAUNCH_CHECK();
  BSB_CUDA(cudaMemsetAsync(out_dir, 0, sizeof(int64_t), s));
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, out_dir + 1, nb, s);
  void* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, tb + 16, s));
  cub::DeviceScan::InclusiveSum(tmp, tb, cnt, out_dir + 1, nb, s);
  BSB_LAUNCH_CHECK();
  const bool shared_dir = col->deep_mode != BSB_DEEP_PACKED;
  const uint8_t* src = col->deep[level - 1];
  vbs_export_level_kernel<<<grid_for(n, 256), 256, 0, s>>>(
      n, level, col->deep_mode, src, col->exist[level - 1], col->exist[1],
      shared_dir ? col->block_dir[1] : col->block_dir[level - 1], out_dir, out_bytes);
  BSB_LAUNCH_CHECK();
  BSB_CUDA(cudaFreeAsync(tmp, s));
  BSB_CUDA(cudaFreeAsync(cnt, s));
  return BSB_OK;
}
