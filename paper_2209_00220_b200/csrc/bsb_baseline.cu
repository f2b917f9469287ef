// bsb_baseline.cu -- the paper's comparison layouts on the device (SURVEY.md
// §8(f) row 4): Bit-Packed (reference bitpacked.py) and VBP / PE-VBP
// (reference vbp.py).  They exist to reproduce the four-layout sweeps, so the
// kernels are straightforward: correct first, HBM-friendly where it is free.
//
// Bit-Packed: code i occupies stream bits [i*w, (i+1)*w), most significant
// bit first, bytes in stream order (bitpacked.py:1-6).  32 rows = 4w bytes =
// w 32-bit words, so one thread owns one output word: it stages its w words
// (byte-swapped to big-endian) in shared memory and extracts 32 codes.  No
// early stop (bitpacked.py:97).
//
// VBP: plane j (j = 0 = most significant bit) is one uint32 per 32-row block
// (bit i = row 32b+i, vbp.py:31-37).  One thread per block walks the planes
// top down with the reference's greater / still-equal masks and stops when
// nothing is still equal (vbp.py:122-141); the PE-VBP variant aligns the
// literal to the padded width (vbp.py:94-98).
#include <cstring>

#include "bsb_common.cuh"

namespace bsb {

constexpr int kBpThreads = 128;

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// ------------------------------------------------------------ Bit-Packed
__global__ void bp_build_kernel(const int64_t* __restrict__ codes, int64_t n, int w,
                                uint32_t* __restrict__ out, int64_t ngroups,
                                unsigned int* __restrict__ err) {
  const uint64_t lim = w >= 64 ? ~0ull : (1ull << w);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint64_t acc = 0;
    int bits = 0;
    int k = 0;
    uint32_t* dst = out + g * w;
    for (int i = 0; i < 32; ++i) {
      const int64_t r = g * 32 + i;
      uint64_t c = 0;
      if (r < n) {
        c = (uint64_t)codes[r];
        if (c >= lim) atomicOr(err, 1u);
        c &= lim - 1;
      }
      acc = (acc << w) | c;
      bits += w;
      if (bits >= 32) {
        bits -= 32;
        dst[k++] = bswap32((uint32_t)(acc >> bits));
        acc &= (1ull << bits) - 1ull;
      }
    }
  }
}

template <bool MASKED>
__global__ void __launch_bounds__(kBpThreads) bp_scan_kernel(
    const uint32_t* __restrict__ words, int64_t n, int64_t ngroups, int w, int op,
    uint64_t lo, uint64_t hi, const uint32_t* __restrict__ mask, uint32_t* __restrict__ out,
    unsigned long long* __restrict__ count) {
  __shared__ uint32_t stage[kBpThreads][33];
  uint32_t* my = stage[threadIdx.x];
  const uint64_t m = (w >= 64) ? ~0ull : ((1ull << w) - 1ull);
  unsigned long long cnt = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < ngroups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* src = words + g * w;
    for (int k = 0; k < w; ++k) my[k] = bswap32(__ldg(src + k));
    my[w] = 0;
    uint32_t res = 0;
    for (int i = 0; i < 32; ++i) {
      const int bp = i * w;
      const int k = bp >> 5, off = bp & 31;
      const uint64_t win = ((uint64_t)my[k] << 32) | my[k + 1];
      const uint64_t v = (win >> (64 - w - off)) & m;
      bool f;
      switch (op) {
        case BSB_EQ: f = v == lo; break;
        case BSB_NE: f = v != lo; break;
        case BSB_LT: f = v < lo; break;
        case BSB_LE: f = v <= lo; break;
        case BSB_GT: f = v > lo; break;
        case BSB_GE: f = v >= lo; break;
        default: f = v >= lo && v <= hi; break;  // BETWEEN (bitpacked.py:90-91)
      }
      res |= (uint32_t)f << i;
    }
    res &= tail_valid(g, n);
    if (MASKED) res &= __ldg(mask + g);  // post-AND (bitpacked.py:113)
    out[g] = res;
    cnt += __popc(res);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(kFull, cnt, d);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(count, cnt);
}

// ------------------------------------------------------------------- VBP
// warp per block: lane = row, one ballot per plane
__global__ void vbp_build_kernel(const uint64_t* __restrict__ codes, int64_t n, int w_max,
                                 uint32_t* __restrict__ planes, int64_t nw,
                                 unsigned int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const uint64_t lim = 1ull << w_max;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nw;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = b * 32 + lane;
    uint64_t c = r < n ? codes[r] : 0ull;
    if (c >= lim) {
      atomicOr(err, 1u);
      c &= lim - 1;
    }
    for (int j = 0; j < w_max; ++j) {
      const uint32_t word = __ballot_sync(kFull, (c >> (w_max - 1 - j)) & 1ull);
      if (lane == 0) planes[(int64_t)j * nw + b] = word;
    }
  }
}

struct VbpLeg {
  uint32_t lit;  // literal aligned to w_max planes
  int op;
};

// One leg over block b (vbp.py:122-141); returns (gt, eq) and the depth.
__device__ __forceinline__ int vbp_leg(const uint32_t* __restrict__ planes, int64_t nw,
                                       int64_t b, int w_max, uint32_t lit, uint32_t valid,
                                       uint32_t& gt, uint32_t& eq,
                                       unsigned long long* words_ctr) {
  uint32_t zeq = valid, zgt = 0;
  int depth = 0;
  for (int j = 0; j < w_max; ++j) {
    if (!zeq) break;
    depth = j + 1;
    if (words_ctr) atomicAdd(words_ctr + j, 1ull);
    const uint32_t d = __ldg(planes + (int64_t)j * nw + b);
    if ((lit >> (w_max - 1 - j)) & 1u) {
      zeq &= d;
    } else {
      zgt |= zeq & d;
      zeq &= ~d;
    }
  }
  gt = zgt;
  eq = zeq;
  return depth;
}

// STATS: counters = int64[2 * BSB_VBP_MAX_PLANES + 2]: words per plane, then
// (bytes are 4 x words), skipped of leg 1, skipped of leg 2.
template <bool BETWEEN, bool STATS>
__global__ void vbp_scan_kernel(const uint32_t* __restrict__ planes, int64_t n, int64_t nw,
                                int w_max, VbpLeg A, VbpLeg B,
                                const uint32_t* __restrict__ mask, uint32_t* __restrict__ out,
                                unsigned long long* __restrict__ count,
                                unsigned long long* __restrict__ stats,
                                int8_t* __restrict__ depth) {
  unsigned long long cnt = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nw;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t valid = tail_valid(b, n);
    if (mask) valid &= __ldg(mask + b);
    uint32_t gt, eq;
    int d = vbp_leg(planes, nw, b, w_max, A.lit, valid, gt, eq, STATS ? stats : nullptr);
    if (STATS && valid == 0) atomicAdd(stats + 2 * 32, 1ull);
    uint32_t res = finalize_op(BETWEEN ? BSB_GE : A.op, gt, eq, valid);
    if (BETWEEN) {
      // leg 2 sees leg 1's result as its input mask (vbp.py:148-151)
      const uint32_t v2 = res;
      const int d2 = vbp_leg(planes, nw, b, w_max, B.lit, v2, gt, eq,
                             STATS ? stats : nullptr);
      if (STATS && v2 == 0) atomicAdd(stats + 2 * 32 + 1, 1ull);
      res = finalize_op(BSB_LE, gt, eq, v2);
      d = d2 > d ? d2 : d;
    }
    out[b] = res;
    if (STATS && depth) depth[b] = (int8_t)d;
    cnt += __popc(res);
  }
#pragma unroll
  for (int dd = 16; dd > 0; dd >>= 1) cnt += __shfl_xor_sync(kFull, cnt, dd);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(count, cnt);
}

// ---------------------------------------------------------------- lookups
__device__ __forceinline__ int64_t decode_plain(const int64_t* values, int64_t n_dict,
                                                const uint64_t* sorted, uint64_t code,
                                                bool& bad) {
  if (sorted) {  // padded prefix-free codes: binary search (dictionary.py:403-411)
    int64_t a = 0, z = n_dict;
    while (a < z) {
      const int64_t mid = (a + z) >> 1;
      if (__ldg(sorted + mid) < code)
        a = mid + 1;
      else
        z = mid;
    }
    if (a >= n_dict || __ldg(sorted + a) != code) {
      bad = true;
      return 0;
    }
    return __ldg(values + a);
  }
  if (code >= (uint64_t)n_dict) {
    bad = true;
    return 0;
  }
  return __ldg(values + code);
}

template <bool VBP>
__global__ void baseline_lookup_kernel(const uint32_t* __restrict__ data, int64_t nw, int w,
                                       const int64_t* __restrict__ rows,
                                       const uint64_t* __restrict__ n_rows_dev,
                                       int64_t n_cap, const int64_t* __restrict__ values,
                                       const uint64_t* __restrict__ sorted, int64_t n_dict,
                                       uint64_t* __restrict__ oc, int64_t* __restrict__ ov,
                                       int32_t* __restrict__ ov32,
                                       unsigned int* __restrict__ err) {
  const int64_t nids = n_rows_dev ? (int64_t)*n_rows_dev : n_cap;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nids;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[i];
    uint64_t code = 0;
    if (VBP) {
      const int64_t b = r >> 5;
      const int bit = (int)(r & 31);
      for (int j = 0; j < w; ++j)
        code = (code << 1) | ((__ldg(data + (int64_t)j * nw + b) >> bit) & 1u);
    } else {
      const int64_t start = r * (int64_t)w;
      const int64_t k = start >> 5;
      const int off = (int)(start & 31);
      const uint64_t win = ((uint64_t)bswap32(__ldg(data + k)) << 32) | bswap32(__ldg(data + k + 1));
      code = (win >> (64 - w - off)) & ((1ull << w) - 1ull);
    }
    if (oc) oc[i] = code;
    if (values) {
      const int64_t v = decode_plain(values, n_dict, sorted, code, bad);
      if (ov) ov[i] = v;
      if (ov32) ov32[i] = (int32_t)v;
    }
  }
  if (bad) atomicOr(err, 1u);
}

static int grid_for(int64_t items, int threads) {
  int64_t g = (items + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

static int check_err(unsigned int* err, cudaStream_t s, int code, const char* msg) {
  unsigned int h = 0;
  BSB_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, s));
  BSB_CUDA(cudaFreeAsync(err, s));
  BSB_CUDA(cudaStreamSynchronize(s));
  if (h) {
    set_error_msg(msg);
    return code;
  }
  return BSB_OK;
}

static int baseline_trivial(int64_t n, int value, const uint32_t* mask, uint32_t* out,
                            uint64_t* count, int64_t* stats, int8_t* depth, cudaStream_t s);

}  // namespace bsb

using namespace bsb;

extern "C" int64_t bsb_bitpacked_words_for(int64_t n_rows, int32_t width_bits) {
  if (n_rows < 0 || width_bits < 1 || width_bits > 32) return -1;
  return ((n_rows + 31) / 32) * width_bits + 2;  // +2: 8-byte lookup window past the end
}

extern "C" int bsb_bitpacked_build(const int64_t* codes, int64_t n, int32_t w, uint32_t* words,
                                   void* stream) {
  if (!codes || !words || n <= 0 || w < 1 || w > 32) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int64_t ng = (n + 31) / 32;
  BSB_CUDA(cudaMemsetAsync(words, 0, (size_t)bsb_bitpacked_words_for(n, w) * 4, s));
  unsigned int* err = nullptr;
  BSB_CUDA(cudaMallocAsync(&err, 4, s));
  BSB_CUDA(cudaMemsetAsync(err, 0, 4, s));
  bp_build_kernel<<<grid_for(ng, 256), 256, 0, s>>>(codes, n, w, words, ng, err);
  BSB_LAUNCH_CHECK();
  return check_err(err, s, BSB_ERANGE, "code out of range for width");
}

extern "C" int bsb_bitpacked_scan(const bsb_bitpacked* col, const bsb_pred* pred,
                                  const uint32_t* mask, uint32_t* out_words, uint64_t* count,
                                  void* stream) {
  if (!col || !pred || !out_words || !count || col->n_rows <= 0 || col->width_bits < 1 ||
      col->width_bits > 32)
    return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  if (pred->trivial >= 0)
    return baseline_trivial(col->n_rows, pred->trivial, mask, out_words, count, nullptr,
                            nullptr, s);
  if (pred->op < BSB_EQ || pred->op > BSB_BETWEEN) return BSB_EINVAL;
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  const int64_t ng = (col->n_rows + 31) / 32;
  auto ull = reinterpret_cast<unsigned long long*>(count);
  const int g = grid_for(ng, kBpThreads);
  if (mask)
    bp_scan_kernel<true><<<g, kBpThreads, 0, s>>>(col->words, col->n_rows, ng, col->width_bits,
                                                  pred->op, pred->code, pred->code2, mask,
                                                  out_words, ull);
  else
    bp_scan_kernel<false><<<g, kBpThreads, 0, s>>>(col->words, col->n_rows, ng,
                                                   col->width_bits, pred->op, pred->code,
                                                   pred->code2, nullptr, out_words, ull);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

extern "C" int bsb_vbp_build(const uint64_t* codes, int64_t n, int32_t w_max, uint32_t* planes,
                             void* stream) {
  if (!codes || !planes || n <= 0 || w_max < 1 || w_max > BSB_VBP_MAX_PLANES) return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int64_t nw = (n + 31) / 32;
  unsigned int* err = nullptr;
  BSB_CUDA(cudaMallocAsync(&err, 4, s));
  BSB_CUDA(cudaMemsetAsync(err, 0, 4, s));
  vbp_build_kernel<<<grid_for(nw * 32, 256), 256, 0, s>>>(codes, n, w_max, planes, nw, err);
  BSB_LAUNCH_CHECK();
  return check_err(err, s, BSB_ERANGE, "code out of range for width");
}

// literal aligned to the planes (vbp.py:94-98): padded encoding shifts the
// prefix-free code (length in bits) up to w_max bits
static bool vbp_literal(const bsb_vbp* col, uint64_t code, int len, uint32_t& lit) {
  if (col->kind == BSB_VBP_PADDED) {
    if (len < 0 || len > col->w_max) return false;
    code <<= (col->w_max - len);
  }
  if (col->w_max < 64 && (code >> col->w_max) != 0) code &= (1ull << col->w_max) - 1ull;
  lit = (uint32_t)code;
  return true;
}

extern "C" int bsb_vbp_scan(const bsb_vbp* col, const bsb_pred* pred, const uint32_t* mask,
                            uint32_t* out_words, uint64_t* count, int64_t* stats, int8_t* depth,
                            void* stream) {
  if (!col || !pred || !out_words || !count || col->n_rows <= 0 || col->w_max < 1 ||
      col->w_max > BSB_VBP_MAX_PLANES)
    return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  if (pred->trivial >= 0)
    return baseline_trivial(col->n_rows, pred->trivial, mask, out_words, count, stats, depth, s);
  if (pred->op < BSB_EQ || pred->op > BSB_BETWEEN) return BSB_EINVAL;
  VbpLeg A, B;
  A.op = pred->op == BSB_BETWEEN ? BSB_GE : pred->op;
  B.op = BSB_LE;
  if (!vbp_literal(col, pred->code, pred->length, A.lit)) return BSB_ERANGE;
  B.lit = 0;
  if (pred->op == BSB_BETWEEN && !vbp_literal(col, pred->code2, pred->length2, B.lit))
    return BSB_ERANGE;
  const int64_t nw = (col->n_rows + 31) / 32;
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  if (stats) BSB_CUDA(cudaMemsetAsync(stats, 0, 8 * BSB_VBP_STATS_WORDS, s));
  auto ull = reinterpret_cast<unsigned long long*>(count);
  auto st = reinterpret_cast<unsigned long long*>(stats);
  const int g = grid_for(nw, 256);
  const bool bt = pred->op == BSB_BETWEEN;
#define BSB_VBP_LAUNCH(BT, ST)                                                                  \
  vbp_scan_kernel<BT, ST><<<g, 256, 0, s>>>(col->planes, col->n_rows, nw, col->w_max, A, B, mask, \
                                            out_words, ull, st, depth)
  if (stats) {
    if (bt) BSB_VBP_LAUNCH(true, true);
    else BSB_VBP_LAUNCH(false, true);
  } else {
    if (bt) BSB_VBP_LAUNCH(true, false);
    else BSB_VBP_LAUNCH(false, false);
  }
#undef BSB_VBP_LAUNCH
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

static int baseline_lookup(bool vbp, const uint32_t* data, int64_t n_rows, int w,
                           const uint32_t* sel_words, const int64_t* rows, int64_t n_ids,
                           const bsb_decode* dec, uint64_t* oc, int64_t* ov, int32_t* ov32,
                           uint64_t* n_out_dev, cudaStream_t s) {
  if (dec && dec->kind != 0 && dec->kind != 1 && dec->kind != 2) return BSB_EINVAL;
  const int64_t* values = (dec && dec->kind) ? dec->values : nullptr;
  const uint64_t* sorted = (dec && dec->kind == 2) ? dec->sorted_padded : nullptr;
  const int64_t n_dict = dec ? dec->n_dict : 0;
  const int64_t nw = (n_rows + 31) / 32;
  int64_t* ids = nullptr;
  uint64_t* cnt = n_out_dev;
  const int64_t cap = sel_words ? n_rows : n_ids;
  if (sel_words) {  // ascending row ids of the selection (bitvector.py:71-72)
    BSB_CUDA(cudaMallocAsync(&ids, (size_t)(n_rows > 0 ? n_rows : 1) * 8, s));
    if (!cnt) BSB_CUDA(cudaMallocAsync(&cnt, 8, s));
    const int rc = bsb_bits_to_rows_async(sel_words, n_rows, 0, ids, cnt, s);
    if (rc) return rc;
  }
  unsigned int* err = nullptr;
  BSB_CUDA(cudaMallocAsync(&err, 4, s));
  BSB_CUDA(cudaMemsetAsync(err, 0, 4, s));
  const int g = grid_for(cap, 256);
  if (vbp)
    baseline_lookup_kernel<true><<<g, 256, 0, s>>>(data, nw, w, sel_words ? ids : rows,
                                                   sel_words ? cnt : nullptr, cap, values,
                                                   sorted, n_dict, oc, ov, ov32, err);
  else
    baseline_lookup_kernel<false><<<g, 256, 0, s>>>(data, nw, w, sel_words ? ids : rows,
                                                    sel_words ? cnt : nullptr, cap, values,
                                                    sorted, n_dict, oc, ov, ov32, err);
  BSB_LAUNCH_CHECK();
  if (ids) BSB_CUDA(cudaFreeAsync(ids, s));
  if (cnt && cnt != n_out_dev) BSB_CUDA(cudaFreeAsync(cnt, s));
  if (!values) {
    BSB_CUDA(cudaFreeAsync(err, s));
    return BSB_OK;
  }
  return check_err(err, s, BSB_ENOTFOUND, "code not in dictionary");
}

extern "C" int bsb_bitpacked_lookup_bits(const bsb_bitpacked* col, const uint32_t* words,
                                         const bsb_decode* dec, uint64_t* out_codes,
                                         int64_t* out_values, int32_t* out_values32,
                                         uint64_t* n_out_dev, void* stream) {
  if (!col || !words || col->n_rows <= 0) return BSB_EINVAL;
  return baseline_lookup(false, col->words, col->n_rows, col->width_bits, words, nullptr, 0,
                         dec, out_codes, out_values, out_values32, n_out_dev,
                         as_stream(stream));
}

extern "C" int bsb_vbp_lookup_bits(const bsb_vbp* col, const uint32_t* words,
                                   const bsb_decode* dec, uint64_t* out_codes,
                                   int64_t* out_values, int32_t* out_values32,
                                   uint64_t* n_out_dev, void* stream) {
  if (!col || !words || col->n_rows <= 0) return BSB_EINVAL;
  return baseline_lookup(true, col->planes, col->n_rows, col->w_max, words, nullptr, 0, dec,
                         out_codes, out_values, out_values32, n_out_dev, as_stream(stream));
}

namespace bsb {
__global__ void baseline_trivial_kernel(int64_t n_rows, int64_t nb, const uint32_t* mask,
                                        int value, uint32_t* out, unsigned long long* count) {
  unsigned long long c = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    if (value) {
      v = tail_valid(b, n_rows);
      if (mask) v &= mask[b];
    }
    out[b] = v;
    c += __popc(v);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// trivial predicates (vbp.py:101-113, bitpacked.py:95-99): every block counts
// as skipped, depth 0
static int baseline_trivial(int64_t n, int value, const uint32_t* mask, uint32_t* out,
                            uint64_t* count, int64_t* stats, int8_t* depth, cudaStream_t s) {
  const int64_t nb = (n + 31) / 32;
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  baseline_trivial_kernel<<<grid_for(nb, 256), 256, 0, s>>>(
      n, nb, mask, value, out, reinterpret_cast<unsigned long long*>(count));
  BSB_LAUNCH_CHECK();
  if (stats) {
    int64_t h[BSB_VBP_STATS_WORDS] = {0};
    h[2 * 32] = nb;
    h[2 * 32 + 1] = nb;
    BSB_CUDA(cudaMemcpyAsync(stats, h, sizeof(h), cudaMemcpyHostToDevice, s));
    BSB_CUDA(cudaStreamSynchronize(s));  // h is a stack buffer
  }
  if (depth) BSB_CUDA(cudaMemsetAsync(depth, 0, nb, s));
  return BSB_OK;
}
}  // namespace bsb
