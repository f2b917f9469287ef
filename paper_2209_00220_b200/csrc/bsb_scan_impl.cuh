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
//
// Latency structure: the caller hands in the tile's level-1 bytes (and for
// PP-VBS the level-2 existence word and tile bases), prefetched one tile
// ahead by the persistent kernels.  Each deeper level costs one dependent
// round trip: its run bytes and the next existence word are issued together.
#pragma once

#include "bsb_common.cuh"

namespace bsb {

struct Leg {
  int32_t len;                 // levels examined (ByteSlice: K; PP-VBS: literal bytes)
  int32_t op;                  // operator when this is the only leg
  PlaneLit pl[kMaxLevels];     // bit-plane carry masks per level (bit-plane blocks)
  LevelLit lv[kMaxLevels];     // byte-split constants (reference-packed deep runs)
  uint32_t byte[kMaxLevels + 1];  // literal byte per level, 0-padded (one spare)
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
  const uint32_t* rexist[kMaxLevels];  // SLICED: deep-row bitmaps of byte j+1
  int32_t K;
  int32_t mode;  // BSB_DEEP_PACKED / BSB_DEEP_SLICED
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

// Level-1 operands of one tile, fetched ahead of use.
struct TileIn {
  uint32_t w[8];   // the lane's 32 swizzled bytes of level 1
  uint32_t m2;     // PP-VBS: existence word of level 2 (every lane)
  int64_t base;    // PP-VBS packed: lane i holds dir[i+2][tile*32]; sliced: dir2[tile*32]
};

__device__ __forceinline__ void fetch_bs(const BsDesc& d, int64_t b, uint32_t valid, TileIn& t) {
  if (valid) {
    ldg256(d.slices + b * 32, t.w);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) t.w[i] = 0;
  }
}

__device__ __forceinline__ void fetch_vbs(const VbsDesc& d, int64_t tile, int64_t b,
                                          uint32_t valid, TileIn& t) {
  const int lane = threadIdx.x & 31;
  if (valid) {
    ldg256(d.bs1 + b * 32, t.w);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) t.w[i] = 0;
  }
  t.m2 = d.K >= 2 ? __ldg(d.exist[1] + b) : 0u;
  if (d.mode != BSB_DEEP_PACKED)
    t.base = d.K >= 2 ? __ldg(d.dir[1] + tile * 32) : 0;
  else
    t.base = (lane + 2 <= d.K) ? __ldg(d.dir[lane + 1] + tile * 32) : 0;
}

// ---------------------------------------------------------------- ByteSlice
// One tile: lane b compares its block level by level (byteslice.py:86-106):
// the level-j sector is loaded only while the block still has tied rows,
// and the warp stops once no lane has one.  Levels are unrolled so every
// literal mask is a constant-bank operand of its LOP3.
template <bool BETWEEN, bool STATS>
__device__ __forceinline__ uint32_t scan_tile_bs(const BsDesc& d, const Leg& A, const Leg& B,
                                                 int64_t b, uint32_t valid, const TileIn& in,
                                                 StatAcc* st, int* depth_out) {
  uint32_t zeqA = valid, zgtA = 0, zeqB = valid, zgtB = 0;
  int depth = 0;
  // level 1: every lane, branch free (invalid lanes carry zero state)
  {
    uint32_t gA, eA, gB, eB;
    if (BETWEEN) {
      cmp_block2(in.w, A.pl[0], B.pl[0], gA, eA, gB, eB);
    } else {
      cmp_block(in.w, A.pl[0], gA, eA);
    }
    if (STATS && valid) {
      depth = 1;
      stat_level<STATS>(st, 0, 32);
    }
    zgtA = zeqA & gA;
    zeqA &= eA & ~gA;
    if (BETWEEN) {
      zgtB = zeqB & gB;
      zeqB &= eB & ~gB & (zeqA | zgtA);  // drop lanes already known to fail GE(lo)
    }
  }
  const uint8_t* base = d.slices + b * 32;
#pragma unroll
  for (int j = 1; j < kMaxLevels; ++j) {
    if (j >= d.K) break;
    const bool act = BETWEEN ? ((zeqA | zeqB) != 0) : (zeqA != 0);
    if (!__any_sync(kFull, act)) break;
    if (act) {
      uint32_t w[8];
      ldg256(base + (int64_t)j * d.stride, w);
      depth = j + 1;
      stat_level<STATS>(st, j, 32);
      if (BETWEEN) {
        uint32_t gA, eA, gB, eB;
        cmp_block2(w, A.pl[j], B.pl[j], gA, eA, gB, eB);
        zgtA |= zeqA & gA;
        zeqA &= eA & ~gA;
        zgtB |= zeqB & gB;
        zeqB &= eB & ~gB & (zeqA | zgtA);
      } else {
        uint32_t g, e;
        cmp_block(w, A.pl[j], g, e);
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
// Works on row-space masks and, unchanged, on packed deep-row masks.
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

// Packed bytes [start, start+cnt) of one block: up to five 8-byte aligned
// loads, then byte alignment with PRMT on demand.
struct Run {
  uint32_t u[10];
  uint32_t sel;
  int qs;
};
__device__ __forceinline__ void load_run(const uint8_t* deep, int64_t start, int cnt, bool act,
                                         Run& r) {
  const uint64_t* p = reinterpret_cast<const uint64_t*>(deep + (start & ~int64_t(7)));
  const int o = (int)(start & 7);
  const int nld = act ? ((o + cnt + 7) >> 3) : 0;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const uint64_t v = (k < nld) ? __ldg(p + k) : 0ull;
    r.u[2 * k] = (uint32_t)v;
    r.u[2 * k + 1] = (uint32_t)(v >> 32);
  }
  r.qs = o >> 2;
  r.sel = 0x3210u + 0x1111u * (uint32_t)(o & 3);
}
__device__ __forceinline__ uint32_t run_word(const Run& r, int i) {
  const uint32_t a = r.qs ? r.u[i + 1] : r.u[i];
  const uint32_t b = r.qs ? r.u[i + 2] : r.u[i + 1];
  return __byte_perm(a, b, r.sel);
}

// Packed compare of a run (nwmax uniform words) against one or two literal
// bytes; bits >= cnt are garbage and masked by the caller.
template <bool TWO>
__device__ __forceinline__ void cmp_run(const Run& r, int nwmax, LevelLit A, LevelLit B,
                                        uint32_t& gA, uint32_t& eA, uint32_t& gB,
                                        uint32_t& eB) {
  uint32_t ga = 0, ea = 0, gb = 0, eb = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i >= nwmax) break;
    const uint32_t w = run_word(r, i);
    const uint32_t ev = __byte_perm(w, 0, 0x4240);
    const uint32_t od = __byte_perm(w, 0, 0x4341);
    ga |= nib4(__byte_perm(ev + A.cgt, od + A.cgt, 0x7351)) << (4 * i);
    ea |= nib4(__byte_perm(ev + A.cge, od + A.cge, 0x7351)) << (4 * i);
    if (TWO) {
      gb |= nib4(__byte_perm(ev + B.cgt, od + B.cgt, 0x7351)) << (4 * i);
      eb |= nib4(__byte_perm(ev + B.cge, od + B.cge, 0x7351)) << (4 * i);
    }
  }
  gA = ga;
  eA = ea & ~ga;
  if (TWO) {
    gB = gb;
    eB = eb & ~gb;
  } else {
    gB = ga;
    eB = eA;
  }
}

// Level 1 of PP-VBS (all lanes, branch free) + its transitions.
template <bool BETWEEN, bool STATS>
__device__ __forceinline__ void vbs_level1(const Leg& A, const Leg& B, int K, uint32_t valid,
                                           const TileIn& in, uint32_t& zeqA, uint32_t& zgtA,
                                           uint32_t& eqfA, uint32_t& zeqB, uint32_t& zgtB,
                                           uint32_t& eqfB, StatAcc* st, int& depth) {
  uint32_t gA, eA, gB, eB;
  if (BETWEEN && A.byte[0] != B.byte[0]) {
    cmp_block2(in.w, A.pl[0], B.pl[0], gA, eA, gB, eB);
  } else {
    cmp_block(in.w, A.pl[0], gA, eA);
    gB = gA;
    eB = eA;
  }
  eA &= ~gA;
  eB &= ~gB;
  if (STATS && valid) {
    depth = 1;
    stat_level<STATS>(st, 0, 32);
  }
  vbs_transition(1, A.len, K, gA, eA, in.m2, zeqA, zgtA, eqfA);
  if (BETWEEN) {
    vbs_transition(1, B.len, K, gB, eB, in.m2, zeqB, zgtB, eqfB);
    zeqB &= zeqA | zgtA | eqfA;
  }
}

// PP-VBS, deep slices in reference packing (one expand per level).
template <bool BETWEEN, bool STATS>
__device__ __forceinline__ uint32_t scan_tile_vbs_packed(const VbsDesc& d, const Leg& A,
                                                         const Leg& B, int64_t tile, int64_t b,
                                                         uint32_t valid, const TileIn& in,
                                                         StatAcc* st, int* depth_out) {
  const int K = d.K;
  uint32_t zeqA = valid, zgtA = 0, eqfA = 0;
  uint32_t zeqB = valid, zgtB = 0, eqfB = 0;
  const int maxlen = BETWEEN ? (A.len > B.len ? A.len : B.len) : A.len;
  int depth = 0;
  vbs_level1<BETWEEN, STATS>(A, B, K, valid, in, zeqA, zgtA, eqfA, zeqB, zgtB, eqfB, st, depth);
  uint32_t mcur = in.m2;
  for (int j = 2; j <= maxlen; ++j) {
    const bool act = BETWEEN ? ((zeqA | zeqB) != 0) : (zeqA != 0);
    if (!__any_sync(kFull, act)) break;
    const int cnt = __popc(mcur);
    const uint32_t incl = warp_incl_scan((uint32_t)cnt);
    const int64_t start = __shfl_sync(kFull, in.base, j - 2) + (int64_t)(incl - cnt);
    Run run;
    load_run(d.deep[j - 1], start, cnt, act, run);
    const uint32_t nxt = (j < K) ? __ldg(d.exist[j] + b) : 0u;
    const int nwmax = __reduce_max_sync(kFull, act ? ((cnt + 3) >> 2) : 0);
    uint32_t pgA, peA, pgB, peB;
    if (BETWEEN && A.byte[j - 1] != B.byte[j - 1])
      cmp_run<true>(run, nwmax, A.lv[j - 1], B.lv[j - 1], pgA, peA, pgB, peB);
    else
      cmp_run<false>(run, nwmax, A.lv[j - 1], A.lv[j - 1], pgA, peA, pgB, peB);
    const uint32_t lowm = cnt >= 32 ? kFull : ((1u << cnt) - 1u);
    const ExpandNet net = expand_setup(mcur);
    const uint32_t gA = expand_apply(net, pgA & lowm), eA = expand_apply(net, peA & lowm);
    uint32_t gB = gA, eB = eA;
    if (BETWEEN) {
      gB = expand_apply(net, pgB & lowm);
      eB = expand_apply(net, peB & lowm);
    }
    if (act) {
      depth = j;
      stat_level<STATS>(st, j - 1, cnt);
    }
    vbs_transition(j, A.len, K, gA, eA, nxt, zeqA, zgtA, eqfA);
    if (BETWEEN) {
      vbs_transition(j, B.len, K, gB, eB, nxt, zeqB, zgtB, eqfB);
      zeqB &= zeqA | zgtA | eqfA;
    }
    mcur = nxt;
  }
  if (STATS) *depth_out = depth;
  if (BETWEEN) return valid & (zgtA | eqfA) & ~zgtB;
  return finalize_op(A.op, zgtA, eqfA, valid);
}

// PP-VBS scan of one tile for the reference-packed deep layout
// (BSB_DEEP_PACKED).  SLICED columns run their own kernels (bsb_vbs_ds.cu,
// bsb_vbs_sliced.cu; stats: bsb_vbs_rows.cu).
template <bool BETWEEN, bool STATS>
__device__ __forceinline__ uint32_t scan_tile_vbs(const VbsDesc& d, const Leg& A,
                                                  const Leg& B, int64_t tile, int64_t b,
                                                  uint32_t valid, const TileIn& in,
                                                  StatAcc* st, int* depth_out) {
  return scan_tile_vbs_packed<BETWEEN, STATS>(d, A, B, tile, b, valid, in, st, depth_out);
}

}  // namespace bsb
