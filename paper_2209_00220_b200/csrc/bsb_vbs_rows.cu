// bsb_vbs_rows.cu -- row-parallel PP-VBS scan of a SLICED column with
// ScanStats (the stats path of bsb_vbs_scan for that layout).
//
// One warp per 32-row block, one lane per row: the lane rebuilds its code's
// bytes (level 1 from the swizzled first slice, deeper levels from the deep
// rows' byte planes) and runs the reference's per-row state machine
// (vbs.py:241-284): compare level by level, drop a tied row that has no next
// byte, settle a tie at the literal's last byte with the existence shortcut.
// The block depth is the warp max of the levels each row stayed tied, which
// gives ScanStats exactly (stats.py:18-45).
#include <cstring>

#include "bsb_scan_impl.cuh"

namespace bsb {

struct RowLeg {
  int32_t len;
  int32_t op;
  uint32_t byte[kMaxLevels];
};

struct RowArgs {
  VbsDesc d;
  int64_t n_rows, nb;
  RowLeg L;
  const uint32_t* mask;
  uint32_t* out;
  unsigned long long* count;
  int64_t* stats;      // may be null
  int8_t* depth;       // may be null
  int32_t skipped_slot;
  int32_t depth_max;
};

// byte j of deep row q (SLICED: bit-plane 32-deep-row blocks)
__device__ __forceinline__ uint32_t plane_byte(const VbsDesc& d, int64_t q, int j) {
  return bp_row_byte(d.deep[j - 1] + (q >> 5) * 32, (int)(q & 31));
}

__global__ void __launch_bounds__(256) vbs_rowscan_kernel(const __grid_constant__ RowArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const VbsDesc& d = a.d;
  const int K = d.K;
  const int l = a.L.len;
  unsigned long long cnt = 0;
  long long words[kMaxLevels] = {0}, bytes[kMaxLevels] = {0}, skipped = 0;
  for (int64_t b = warp; b < a.nb; b += nwarps) {
    uint32_t valid = tail_valid(b, a.n_rows);
    if (a.mask) valid &= __ldg(a.mask + b);
    const bool v = (valid >> lane) & 1u;
    int t = 0;
    bool gt = false, eq = false;
    uint32_t m[kMaxLevels];
    int len = 1;
#pragma unroll
    for (int j = 2; j <= kMaxLevels; ++j) {
      m[j - 1] = (j <= K) ? __ldg(d.exist[j - 1] + b) : 0u;
      len += (j <= K) && ((m[j - 1] >> lane) & 1u);
    }
    if (v) {
      const uint32_t below = (1u << lane) - 1u;
      const int64_t q = K >= 2 ? __ldg(d.dir[1] + b) + __popc(m[1] & below) : 0;
      t = 1;
      for (int j = 1;; ++j) {
        const uint32_t cj = j == 1 ? bp_row_byte(d.bs1 + b * 32, lane)
                                   : plane_byte(d, q, j);
        const uint32_t lj = a.L.byte[j - 1];
        if (cj != lj) {
          gt = cj > lj;
          break;
        }
        if (j < l) {
          if (len > j) {
            t = j + 1;
            continue;
          }
          break;  // shorter code with an equal prefix: less
        }
        if (l < K && len > l)
          gt = true;  // existence shortcut (vbs.py:276-280)
        else
          eq = true;
        break;
      }
    }
    const uint32_t gw = __ballot_sync(kFull, gt), ew = __ballot_sync(kFull, eq);
    const int depth = __reduce_max_sync(kFull, (unsigned)t);
    const uint32_t res = finalize_op(a.L.op, gw, ew, valid);
    if (lane == 0) {
      a.out[b] = res;
      if (a.depth) {
        if (a.depth_max) {
          const int8_t old = a.depth[b];
          a.depth[b] = (int8_t)(depth > old ? depth : old);
        } else {
          a.depth[b] = (int8_t)depth;
        }
      }
      cnt += __popc(res);
      if (a.stats) {
        skipped += valid == 0;
#pragma unroll
        for (int j = 1; j <= kMaxLevels; ++j) {
          if (j <= depth) {
            words[j - 1] += 1;
            bytes[j - 1] += j == 1 ? 32 : __popc(m[j - 1]);
          }
        }
      }
    }
  }
  if (lane == 0) {
    if (cnt) atomicAdd(a.count, cnt);
    if (a.stats) {
      for (int j = 0; j < kMaxLevels; ++j) {
        if (words[j]) atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + j),
                                (unsigned long long)words[j]);
        if (bytes[j]) atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + 8 + j),
                                (unsigned long long)bytes[j]);
      }
      if (skipped)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + a.skipped_slot),
                  (unsigned long long)skipped);
    }
  }
}

static void row_leg(RowLeg& L, int op, uint64_t code, int len) {
  std::memset(&L, 0, sizeof(L));
  L.op = op;
  L.len = len;
  for (int j = 0; j < len && j < kMaxLevels; ++j)
    L.byte[j] = (uint32_t)((code >> (8 * (len - 1 - j))) & 0xFF);
}

static int launch_rows(const RowArgs& a, cudaStream_t s) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vbs_rowscan_kernel, 256, 0);
  int64_t want = (a.nb + 7) / 8;
  int64_t cap = (int64_t)sm_count() * (per_sm > 0 ? per_sm : 1);
  int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  vbs_rowscan_kernel<<<grid, 256, 0, s>>>(a);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

// Scan of a SLICED column through the row-parallel kernel.  BETWEEN runs as
// the reference's two pipelined legs (vbs.py:299-304); with `stats` the
// counters follow stats.py:47-67 (slots 17/19 hold the legs' skipped blocks).
int vbs_rows_scan(const VbsDesc& d, int64_t n_rows, const bsb_pred* p, const uint32_t* mask,
                  uint32_t* out, uint64_t* count, int64_t* stats, int8_t* depth,
                  cudaStream_t s) {
  RowArgs a;
  std::memset(&a, 0, sizeof(a));
  a.d = d;
  a.n_rows = n_rows;
  a.nb = (n_rows + 31) / 32;
  a.mask = mask;
  a.stats = stats;
  a.depth = depth;
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  if (stats) {
    int64_t h[BSB_STATS_WORDS] = {0};
    h[16] = a.nb;
    h[18] = d.K;
    BSB_CUDA(cudaMemcpyAsync(stats, h, sizeof(h), cudaMemcpyHostToDevice, s));
  }
  if (p->op != BSB_BETWEEN) {
    row_leg(a.L, p->op, p->code, p->length);
    a.out = out;
    a.count = reinterpret_cast<unsigned long long*>(count);
    a.skipped_slot = 17;
    int rc = launch_rows(a, s);
    if (stats) BSB_CUDA(cudaStreamSynchronize(s));
    return rc;
  }
  uint32_t* tmp = nullptr;
  unsigned long long* dummy = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, (size_t)a.nb * 4 + 4, s));
  BSB_CUDA(cudaMallocAsync(&dummy, 8, s));
  BSB_CUDA(cudaMemsetAsync(dummy, 0, 8, s));
  RowArgs l1 = a;
  row_leg(l1.L, BSB_GE, p->code, p->length);
  l1.out = tmp;
  l1.count = dummy;
  l1.skipped_slot = 17;
  int rc = launch_rows(l1, s);
  if (rc) return rc;
  RowArgs l2 = a;
  row_leg(l2.L, BSB_LE, p->code2, p->length2);
  l2.mask = tmp;
  l2.out = out;
  l2.count = reinterpret_cast<unsigned long long*>(count);
  l2.skipped_slot = 19;
  l2.depth_max = 1;
  rc = launch_rows(l2, s);
  if (rc) return rc;
  BSB_CUDA(cudaFreeAsync(tmp, s));
  BSB_CUDA(cudaFreeAsync(dummy, s));
  if (stats) BSB_CUDA(cudaStreamSynchronize(s));
  return BSB_OK;
}

}  // namespace bsb
