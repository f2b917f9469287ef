// bsb_scan_impl.cuh -- warp-collective tile scans for ByteSlice and PP-VBS.
//
// A warp scans one tile (32 blocks x 32 rows); lane b owns block b.  Every
// lane of the warp must call the tile functions together (they use shuffles
// and votes); lanes whose block is outside the column pass valid == 0.
//
// Semantics follow the reference exactly:
//   ByteSlice  byteslice.py:76-106  (GT/EQ state machine per byte plane)
//   PP-VBS     vbs.py:222-289       (Alg. 3, existence shortcut)
//   finalize   vbs.py:179-197
// A fused BETWEEN evaluates GE(lo) and LE(hi) in one pass over the slices;
// the result equals the reference's pipelined legs (vbs.py:299-304) because
// hi-leg lanes are only dropped once they are known to fail the lo leg.
#pragma once

#include "bsb_common.cuh"

namespace bsb {

struct Leg {
  int32_t len;                 // levels examined (ByteSlice: K; PP-VBS: literal bytes)
  int32_t op;                  // operator when this is the only leg
  LevelLit lv[kMaxLevels];
  uint32_t byte[kMaxLevels];   // literal byte per level (for same-byte sharing)
};

struct BsDesc {
  const uint8_t* slices;
  int64_t stride;
  int32_t K;
};

struct VbsDesc {
  const uint8_t* bs1;
  const uint8_t* deep[kMaxLevels];
  const uint32_t* exist[kMaxLevels];
  const int64_t* dir[kMaxLevels];
  int32_t K;
};

// Per-lane statistics accumulators (reference stats.py:18-45).
struct StatAcc {
  int64_t words[kMaxLevels];
  int64_t bytes[kMaxLevels];
  int64_t skipped;
};

template <bool STATS>
__device__ __forceinline__ void stat_level(StatAcc* st, int j, int64_t nbytes) {
  if (STATS) {
    st->words[j] += 1;
    st->bytes[j] += nbytes;
  }
}

// ---------------------------------------------------------------- ByteSlice
// Returns the lane's result word.  `depth_out` (STATS) = deepest level loaded.
template <bool BETWEEN, bool STATS>
__device__ __forceinline__ uint32_t scan_tile_bs(const BsDesc& d, const Leg& A, const Leg& B,
                                                 int64_t b, uint32_t valid, StatAcc* st,
                                                 int* depth_out) {
  uint32_t zeqA = valid, zgtA = 0, zeqB = valid, zgtB = 0;
  int depth = 0;
  const uint8_t* base = d.slices + b * 32;
  for (int j = 0; j < d.K; ++j) {
    const bool act = BETWEEN ? ((zeqA | zeqB) != 0) : (zeqA != 0);
    if (!__any_sync(kFull, act)) break;
    if (act) {
      uint32_t w[8];
      ldg256(base + (int64_t)j * d.stride, w);
      depth = j + 1;
      stat_level<STATS>(st, j, 32);
      if (BETWEEN) {
        uint32_t gA, eA, gB, eB;
        if (A.byte[j] == B.byte[j]) {
          cmp_block(w, A.lv[j], gA, eA);
          gB = gA;
          eB = eA;
        } else {
          cmp_block2(w, A.lv[j], B.lv[j], gA, eA, gB, eB);
        }
        eA &= ~gA;
        eB &= ~gB;
        zgtA |= zeqA & gA;
        zeqA &= eA;
        zgtB |= zeqB & gB;
        zeqB &= eB & (zeqA | zgtA);  // drop lanes already known to fail GE(lo)
      } else {
        uint32_t g, e;
        cmp_block(w, A.lv[j], g, e);
        zgtA |= zeqA & g;
        zeqA &= e & ~g;
      }
    }
  }
  if (STATS) *depth_out = depth;
  if (BETWEEN) return valid & (zgtA | zeqA) & ~zgtB;
  return finalize_op(A.op, zgtA, zeqA, valid);
}

// ------------------------------------------------------------------ PP-VBS
// Transition after comparing level j (1-based) -- reference vbs.py:272-284.
__device__ __forceinline__ void vbs_transition(int j, int len, int K, uint32_t g, uint32_t e,
                                               uint32_t nxt, uint32_t& zeq, uint32_t& zgt,
                                               uint32_t& eqf) {
  if (j > len) return;
  if (j < len) {
    zgt |= zeq & g;
    zeq = zeq & e & nxt;
  } else if (len < K) {
    const uint32_t still = zeq & e;
    zgt |= (zeq & g) | (still & nxt);  // longer code, equal prefix => greater
    eqf = still & ~nxt;
    zeq = 0;
  } else {
    zgt |= zeq & g;
    eqf = zeq & e;
    zeq = 0;
  }
}

// Load the packed level bytes [start, start+cnt) of one block as u32 words.
__device__ __forceinline__ void load_run(const uint8_t* deep, int64_t start, int cnt,
                                         uint32_t (&R)[8]) {
  const uint64_t* p = reinterpret_cast<const uint64_t*>(deep + (start & ~int64_t(7)));
  const int o = (int)(start & 7);
  const int nld = (o + cnt + 7) >> 3;
  uint64_t q[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) q[k] = (k < nld) ? __ldg(p + k) : 0ull;
  const unsigned sh = 8u * o;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t v = sh ? ((q[i] >> sh) | (q[i + 1] << (64u - sh))) : q[i];
    R[2 * i] = (uint32_t)v;
    R[2 * i + 1] = (uint32_t)(v >> 32);
  }
}

template <bool BETWEEN, bool STATS>
__device__ __forceinline__ uint32_t scan_tile_vbs(const VbsDesc& d, const Leg& A,
                                                  const Leg& B, int64_t tile, int64_t b,
                                                  uint32_t valid, StatAcc* st,
                                                  int* depth_out) {
  const int K = d.K;
  uint32_t zeqA = valid, zgtA = 0, eqfA = 0;
  uint32_t zeqB = valid, zgtB = 0, eqfB = 0;
  const int maxlen = BETWEEN ? (A.len > B.len ? A.len : B.len) : A.len;
  int depth = 0;
  uint32_t mcur = 0;  // existence word of the current level (all lanes)

  for (int j = 1; j <= maxlen; ++j) {
    const bool act = BETWEEN ? ((zeqA | zeqB) != 0) : (zeqA != 0);
    if (!__any_sync(kFull, act)) break;
    uint32_t gA = 0, eA = 0, gB = 0, eB = 0;
    if (j == 1) {
      if (act) {
        uint32_t w[8];
        ldg256(d.bs1 + b * 32, w);
        depth = 1;
        stat_level<STATS>(st, 0, 32);
        if (BETWEEN && A.byte[0] != B.byte[0]) {
          cmp_block2(w, A.lv[0], B.lv[0], gA, eA, gB, eB);
        } else {
          cmp_block(w, A.lv[0], gA, eA);
          gB = gA;
          eB = eA;
        }
        eA &= ~gA;
        eB &= ~gB;
      }
    } else {
      // bytes of this block at level j: BS_j[dir_j[tile*32] + prefix .. + cnt)
      const int cnt = __popc(mcur);
      const uint32_t incl = warp_incl_scan((uint32_t)cnt);
      const int64_t base = __ldg(d.dir[j - 1] + tile * 32);
      const int64_t start = base + (int64_t)(incl - cnt);
      const int nw = (cnt + 3) >> 2;
      const int nwmax = __reduce_max_sync(kFull, act ? nw : 0);
      if (act) {
        depth = j;
        stat_level<STATS>(st, j - 1, cnt);
        uint32_t R[8];
        load_run(d.deep[j - 1], start, cnt, R);
        uint32_t pgA = 0, peA = 0, pgB = 0, peB = 0;
        const bool same = !BETWEEN || (A.byte[j - 1] == B.byte[j - 1]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < nwmax) {
            uint32_t g4, e4;
            cmp_word_packed(R[i], A.lv[j - 1], g4, e4);
            pgA |= g4 << (4 * i);
            peA |= e4 << (4 * i);
            if (BETWEEN && !same) {
              cmp_word_packed(R[i], B.lv[j - 1], g4, e4);
              pgB |= g4 << (4 * i);
              peB |= e4 << (4 * i);
            }
          }
        }
        const uint32_t lowm = cnt >= 32 ? kFull : ((1u << cnt) - 1u);
        pgA &= lowm;
        peA &= lowm & ~pgA;
        const ExpandNet net = expand_setup(mcur);
        gA = pgA ? expand_apply(net, pgA) : 0u;
        eA = peA ? expand_apply(net, peA) : 0u;
        if (BETWEEN) {
          if (same) {
            gB = gA;
            eB = eA;
          } else {
            pgB &= lowm;
            peB &= lowm & ~pgB;
            gB = pgB ? expand_apply(net, pgB) : 0u;
            eB = peB ? expand_apply(net, peB) : 0u;
          }
        }
      }
    }
    // existence word of level j+1 for every lane (transition + next prefix)
    uint32_t nxt = 0;
    if (j < K) {
      const uint32_t* ex = d.exist[j];
      nxt = (valid != 0 || true) ? __ldg(ex + b) : 0u;
    }
    if (act) {
      vbs_transition(j, A.len, K, gA, eA, nxt, zeqA, zgtA, eqfA);
      if (BETWEEN) {
        vbs_transition(j, B.len, K, gB, eB, nxt, zeqB, zgtB, eqfB);
        zeqB &= zeqA | zgtA | eqfA;  // drop lanes known to fail GE(lo)
      }
    }
    mcur = nxt;
  }
  if (STATS) *depth_out = depth;
  if (BETWEEN) return valid & (zgtA | eqfA) & ~zgtB;
  return finalize_op(A.op, zgtA, eqfA, valid);
}

}  // namespace bsb
