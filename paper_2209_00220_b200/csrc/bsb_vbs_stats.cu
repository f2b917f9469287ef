// bsb_vbs_stats.cu -- ScanStats of a SLICED PP-VBS scan in deep-row space.
//
// The reference's ScanStats (stats.py:18-84, vbs.py:286-287) are block
// counters of its early-stopping scan: a block is active at level j while it
// has rows tied with the literal entering level j.  A row's own depth is
// 1 + the number of Alg. 3 transitions it survives (vbs.py:272-284: tied on
// bytes 1..j and owning byte j+1); a block's depth is the maximum over its
// valid rows.  This kernel runs the deep-space scan of vbs_ds_kernel (phase 1
// shallow rows by byte thresholds, phase 2 the deep rows level by level in
// 32-deep-row blocks, phase 3 back to row space) and additionally carries each
// deep row's survival count as three bit planes, deposits them at the rows'
// M_2 lanes (pdep) and takes the bit-sliced maximum over the block's valid
// rows -- the block depth -- from which the level counters follow.  BETWEEN
// emulates the reference's two pipelined legs (vbs.py:299-304): leg 2 counts
// only rows passing GE(lo), and its tie tracking is not pruned by leg 1.
// Replaces the row-parallel stats kernel (bsb_vbs_rows.cu) for columns the
// deep-space kernel can scan; results words and counts are the same as the
// plain scan's.
#include <cstdlib>
#include <cstring>

#include "bsb_scan_impl.cuh"

namespace bsb {

const PdepTables* pdep_tables(cudaStream_t s);  // bsb_vbs_ds.cu

constexpr int kStThreads = 256;
constexpr int kStWarps = kStThreads / 32;

struct DsStatArgs {
  int64_t n_rows, nb, ntiles, nbpad;
  VbsDesc d;
  Leg A, B;
  PlaneThr tP, tQ;
  int twoQ;
  uint32_t inv;
  int d1;
  uint32_t d1gA, d1eA, d1gB, d1eB;
  const uint32_t* mask;
  uint32_t* out;
  unsigned long long* count;
  int64_t* stats;  // int64[24]: words [0..7], bytes [8..15], skipped legs [17] / [19]
  int8_t* depth;   // per block, may be null
  const PdepTables* pdep;
};

__device__ __forceinline__ void set_t(uint32_t S, int j, uint32_t (&T)[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) T[k] = (T[k] & ~S) | (((j >> k) & 1) ? S : 0u);
}

// maximum of the 3-bit values (bit planes R) over the rows in c
__device__ __forceinline__ int max_t(const uint32_t (&R)[3], uint32_t c) {
  int mx = 0;
  if (c) {
    if (R[2] & c) {
      mx |= 4;
      c &= R[2];
    }
    if (R[1] & c) {
      mx |= 2;
      c &= R[1];
    }
    if (R[0] & c) mx |= 1;
  }
  return mx;
}

// One warp per super-tile of ST tiles (as vbs_ds_kernel): phase 1 and 3
// lane = row block of tile u, phase 2 lane = deep block of the super-tile
// (about ST x the deep blocks of one tile per pass: fuller lanes).
template <bool BETWEEN, int ST>
__global__ void __launch_bounds__(kStThreads, 3) vbs_ds_stats_kernel(const __grid_constant__ DsStatArgs a) {
  constexpr int kRd = ST * 32 + 8;  // deep blocks a super-tile touches + guard words
  // per warp: final words, GE(lo) words, survival planes of both legs
  __shared__ uint32_t sm_all[kStWarps][8][kRd];
  uint32_t (*sm)[kRd] = sm_all[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const VbsDesc& d = a.d;
  const int K = d.K;
  const Leg& A = a.A;
  const Leg& B = a.B;
  const int lenA = A.len, lenB = BETWEEN ? B.len : 0;
  const int maxlen = lenA > lenB ? lenA : lenB;
  const int64_t nsuper = (a.ntiles + ST - 1) / ST;
  unsigned long long cnt = 0;
  // per-lane counters (32-bit: a lane sees at most 64 level reads per tile)
  uint32_t words[kMaxLevels], bytes[kMaxLevels], skA = 0, skB = 0;
#pragma unroll
  for (int j = 0; j < kMaxLevels; ++j) words[j] = bytes[j] = 0;
  for (int64_t sp = warp; sp < nsuper; sp += nwarps) {
    const int64_t D0 = K >= 2 ? __ldg(d.dir[1] + (sp * ST * 32 < a.nbpad ? sp * ST * 32 : a.nbpad)) : 0;
    const int sh0 = (int)(D0 & 31);
    // ---- phase 1: shallow rows by byte thresholds (lane = row block)
    uint32_t rs[ST], gs[ST], vs[ST], ms[ST];
    int offs[ST];
    int soff = 0;
#pragma unroll
    for (int u = 0; u < ST; ++u) {
      const int64_t tile = sp * ST + u;
      const int64_t b = tile * 32 + lane;
      const bool in = tile < a.ntiles && b < a.nb;
      uint32_t w[8];
      if (in) {
        ldg256(d.bs1 + b * 32, w);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = 0;
      }
      const uint32_t m2 = (in && K >= 2) ? __ldg(d.exist[1] + b) : 0u;
      uint32_t valid = in ? tail_valid(b, a.n_rows) : 0u;
      if (a.mask && in) valid &= __ldg(a.mask + b);
      const uint32_t P = bp_ge(w, a.tP);
      const uint32_t Q = a.twoQ ? bp_ge(w, a.tQ) : 0u;
      rs[u] = valid & ~m2 & ((P & ~Q) ^ a.inv);
      gs[u] = valid & ~m2 & P;  // BETWEEN: shallow rows passing GE(lo)
      vs[u] = valid;
      ms[u] = m2;
      const int c2 = __popc(m2);
      const uint32_t incl = warp_incl_scan((uint32_t)c2);
      offs[u] = sh0 + soff + (int)(incl - (uint32_t)c2);
      soff += (int)__shfl_sync(kFull, incl, 31);
    }
    const int ndt = (sh0 + soff + 31) >> 5;
    const int64_t db0 = D0 >> 5;
    // ---- phase 2: deep rows, lane = deep block
    for (int t0 = 0; t0 < ndt; t0 += 32) {
      const int t = t0 + lane;
      const bool has = t < ndt;
      const int64_t dbk = db0 + t;
      uint32_t zA = has ? kFull : 0u, zB = (BETWEEN && has) ? kFull : 0u;
      uint32_t gtA = 0, eqA = 0, gtB = 0, eqB = 0;
      uint32_t TA[3] = {0u, 0u, 0u}, TB[3] = {0u, 0u, 0u};
      int j0 = 1;
      if (a.d1) {  // level 1 of the deep rows from the zone map
        vbs_transition(1, lenA, K, a.d1gA, a.d1eA, kFull, zA, gtA, eqA);
        if (1 < lenA) set_t(zA, 1, TA);
        if (BETWEEN) {
          vbs_transition(1, lenB, K, a.d1gB, a.d1eB, kFull, zB, gtB, eqB);
          if (1 < lenB) set_t(zB, 1, TB);
        }
        j0 = 2;
      }
#pragma unroll 1
      for (int j = j0; j <= maxlen; ++j) {
        const bool act = BETWEEN ? ((zA | zB) != 0) : (zA != 0);
        if (!__any_sync(kFull, act)) break;
        uint32_t v[8];
        if (act) {
          if (j >= 3)
            ldg256_sparse(d.deep[j - 1] + dbk * 32, v);
          else
            ldg256(d.deep[j - 1] + dbk * 32, v);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = 0;
        }
        const uint32_t nxt =
            j >= K ? 0u : (j == 1 ? kFull : (act ? __ldg(d.rexist[j] + dbk) : 0u));
        uint32_t gA, gaE, gB, gbE;
        cmp_block(v, A.pl[j - 1], gA, gaE);
        gaE &= ~gA;
        vbs_transition(j, lenA, K, gA, gaE, nxt, zA, gtA, eqA);
        if (j < lenA) set_t(zA, j, TA);
        if (BETWEEN) {
          cmp_block(v, B.pl[j - 1], gB, gbE);
          gbE &= ~gB;
          vbs_transition(j, lenB, K, gB, gbE, nxt, zB, gtB, eqB);
          if (j < lenB) set_t(zB, j, TB);  // pure hi-tie tracking (leg 2 of the pipeline)
        }
      }
      if (has) {
        sm[0][t] = BETWEEN ? ((gtA | eqA) & ~gtB) : finalize_op(A.op, gtA, eqA, kFull);
        sm[1][t] = gtA | eqA;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          sm[2 + k][t] = TA[k];
          sm[5 + k][t] = TB[k];
        }
      }
    }
    if (lane < 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) sm[q][ndt + lane] = 0u;  // guard words
    }
    __syncwarp();
    // ---- phase 3: back to row space (lane = row block)
#pragma unroll
    for (int u = 0; u < ST; ++u) {
      const int64_t b = (sp * ST + u) * 32 + lane;
      const bool in = sp * ST + u < a.ntiles && b < a.nb;
      const uint32_t m2 = ms[u], valid = vs[u];
      const int c2 = __popc(m2);
      const int wi = offs[u] >> 5, sb = offs[u] & 31;
      const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
      auto win = [&](int q) -> uint32_t {
        if (!c2) return 0u;
        const uint32_t x = __funnelshift_r(sm[q][wi], sm[q][wi + 1], sb) & lowm;
        return x == 0u ? 0u : (x == lowm ? m2 : pdep_tab_g(a.pdep, x, m2));
      };
      // raw window of plane q: this block's deep rows in deep-row order
      auto raw = [&](int q) -> uint32_t {
        return c2 ? __funnelshift_r(sm[q][wi], sm[q][wi + 1], sb) & lowm : 0u;
      };
      const uint32_t res = rs[u] | (win(0) & valid);
      uint32_t R[3];
      int dA = 0, dB = 0;
      uint32_t valid2 = 0;
      if (valid == kFull) {
        // every row valid: the depths are maxima over deep-row windows, no
        // deposit needed (valid & M_2 = all of the block's deep rows)
#pragma unroll
        for (int k = 0; k < 3; ++k) R[k] = raw(2 + k);
        dA = 1 + max_t(R, lowm);
        if (BETWEEN) {
          const uint32_t ge_deep = raw(1);  // deep rows passing GE(lo)
          valid2 = gs[u] | ge_deep;         // nonzero iff some row passes
#pragma unroll
          for (int k = 0; k < 3; ++k) R[k] = raw(5 + k);
          dB = valid2 ? 1 + max_t(R, ge_deep) : 0;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) R[k] = win(2 + k) & valid;
        dA = valid ? 1 + max_t(R, valid & m2) : 0;
        if (BETWEEN) {
          valid2 = valid & (gs[u] | (win(1) & m2));
#pragma unroll
          for (int k = 0; k < 3; ++k) R[k] = win(5 + k) & valid2;
          dB = valid2 ? 1 + max_t(R, valid2 & m2) : 0;
        }
      }
      if (in) {
        a.out[b] = res;
        cnt += __popc(res);
        if (a.depth) a.depth[b] = (int8_t)(dA > dB ? dA : dB);
        skA += valid == 0;
        if (BETWEEN) skB += valid2 == 0;
#pragma unroll
        for (int j = 0; j < kMaxLevels; ++j) {
          const uint32_t act = (dA > j) + (BETWEEN ? (dB > j) : 0);
          if (act) {
            words[j] += act;
            bytes[j] += act * (j == 0 ? 32u : (uint32_t)__popc(__ldg(d.exist[j] + b)));
          }
        }
      }
    }
    __syncwarp();
  }
  // warp sums in 64 bits (a warp's total can pass 2^32 on long columns)
  auto wsum = [&](uint32_t v) -> unsigned long long {
    unsigned long long x = v;
#pragma unroll
    for (int dd = 16; dd > 0; dd >>= 1) x += __shfl_xor_sync(kFull, x, dd);
    return x;
  };
#pragma unroll
  for (int dd = 16; dd > 0; dd >>= 1) cnt += __shfl_xor_sync(kFull, cnt, dd);
  unsigned long long* st = reinterpret_cast<unsigned long long*>(a.stats);
#pragma unroll
  for (int j = 0; j < kMaxLevels; ++j) {
    const unsigned long long wj = wsum(words[j]), bj = wsum(bytes[j]);
    if (lane == 0 && wj) atomicAdd(st + j, wj);
    if (lane == 0 && bj) atomicAdd(st + 8 + j, bj);
  }
  const unsigned long long sa = wsum(skA), sbk = BETWEEN ? wsum(skB) : 0ull;
  if (lane == 0) {
    if (cnt) atomicAdd(a.count, cnt);
    if (sa) atomicAdd(st + 17, sa);
    if (BETWEEN && sbk) atomicAdd(st + 19, sbk);
  }
}

// ScanStats path of a SLICED column with deep[0] or the zone map (the
// deep-space kernel's preconditions).  `thr`: the phase-1 thresholds of
// vbs_ds_scan for this predicate.
int vbs_ds_stats_scan(const VbsDesc& d, int64_t n_rows, int64_t stride, int deep1_shared,
                      const Leg& A, const Leg& B, bool between, int tP, int tQ, uint32_t inv,
                      const uint32_t* mask, uint32_t* out, unsigned long long* count,
                      int64_t* stats, int8_t* depth, cudaStream_t s) {
  DsStatArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_rows = n_rows;
  a.nb = (n_rows + 31) / 32;
  a.ntiles = (a.nb + 31) / 32;
  a.nbpad = stride / 32;
  a.d = d;
  a.A = A;
  a.B = B;
  a.tP = make_plane_thr(tP);
  a.tQ = make_plane_thr(tQ);
  a.twoQ = tQ < 256;
  a.inv = inv;
  if (deep1_shared >= 1 && deep1_shared <= 256) {
    const uint32_t x = (uint32_t)(deep1_shared - 1);
    a.d1 = 1;
    a.d1gA = x > A.byte[0] ? kFull : 0u;
    a.d1eA = x == A.byte[0] ? kFull : 0u;
    a.d1gB = x > B.byte[0] ? kFull : 0u;
    a.d1eB = x == B.byte[0] ? kFull : 0u;
  }
  a.mask = mask;
  a.out = out;
  a.count = count;
  a.stats = stats;
  a.depth = depth;
  a.pdep = pdep_tables(s);
  if (!a.pdep) return BSB_ECUDA;
  int64_t h[BSB_STATS_WORDS] = {0};
  h[16] = a.nb;
  h[18] = d.K;
  BSB_CUDA(cudaMemcpyAsync(stats, h, sizeof(h), cudaMemcpyHostToDevice, s));
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  const char* ste = std::getenv("BSB_STATS_ST");
  const int ST = ste ? std::atoi(ste) : 4;
  auto go = [&](auto kern) -> int {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStThreads, 0);
    if (per_sm < 1) per_sm = 1;
    const int64_t nsuper = (a.ntiles + ST - 1) / ST;
    const int64_t want = (nsuper + kStWarps - 1) / kStWarps;
    const int64_t cap = (int64_t)sm_count() * per_sm;
    const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
    kern<<<grid, kStThreads, 0, s>>>(a);
    BSB_LAUNCH_CHECK();
    return BSB_OK;
  };
  // (h is pageable: cudaMemcpyAsync has staged it before returning)
  if (ST == 4) return between ? go(vbs_ds_stats_kernel<true, 4>) : go(vbs_ds_stats_kernel<false, 4>);
  if (ST == 1) return between ? go(vbs_ds_stats_kernel<true, 1>) : go(vbs_ds_stats_kernel<false, 1>);
  return between ? go(vbs_ds_stats_kernel<true, 2>) : go(vbs_ds_stats_kernel<false, 2>);
}

}  // namespace bsb
