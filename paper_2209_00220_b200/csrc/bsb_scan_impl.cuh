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
  LevelLit lv[kMaxLevels];
  uint32_t byte[kMaxLevels + 1];  // literal byte per level, 0-padded (one spare for planes)
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
  const uint32_t* rexist[kMaxLevels];  // PLANES: deep-row bitmaps of byte j+1
  int32_t K;
  int32_t mode;  // BSB_DEEP_PACKED / BSB_DEEP_RANK2 / BSB_DEEP_PLANES
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
  int64_t base;    // PP-VBS packed: lane i holds dir[i+2][tile*32]; rank2: dir2[tile*32]
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
// levels >= 2 where every live block has at most this many tied rows compare
// those rows' bytes one by one instead of the 32-byte SWAR compare
constexpr int kSparseRows = 4;

// L1Z: the (lo) literal's level-1 byte is 0x00 (host-selected variant).
template <bool BETWEEN, bool STATS, bool L1Z = false>
__device__ __forceinline__ uint32_t scan_tile_bs(const BsDesc& d, const Leg& A, const Leg& B,
                                                 int64_t b, uint32_t valid, const TileIn& in,
                                                 StatAcc* st, int* depth_out) {
  uint32_t zeqA = valid, zgtA = 0, zeqB = valid, zgtB = 0;
  int depth = 0;
  // level 1: every lane, branch free (invalid lanes carry zero state)
  {
    uint32_t gA, eA, gB, eB;
    if (BETWEEN && A.byte[0] != B.byte[0]) {
      if (L1Z)
        cmp_block2_z(in.w, A.lv[0], B.lv[0], gA, eA, gB, eB);
      else
        cmp_block2(in.w, A.lv[0], B.lv[0], gA, eA, gB, eB);
    } else {
      if (L1Z)
        cmp_block_z(in.w, A.lv[0], gA, eA);
      else
        cmp_block(in.w, A.lv[0], gA, eA);
      gB = gA;
      eB = eA;
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
  for (int j = 1; j < d.K; ++j) {
    const bool act = BETWEEN ? ((zeqA | zeqB) != 0) : (zeqA != 0);
    if (!__any_sync(kFull, act)) break;
    const uint32_t cand = BETWEEN ? (zeqA | zeqB) : zeqA;
    if (BETWEEN && !STATS && !__any_sync(kFull, __popc(cand) > kSparseRows)) {
      // every live block has only a few tied rows: compare just their bytes
      if (act) {
        uint32_t w[8];
        ldg256(base + (int64_t)j * d.stride, w);
        const uint32_t la = A.byte[j], lb = B.byte[j];
        uint32_t gA = 0, eA = 0, gB = 0, eB = 0;
        for (uint32_t rest = cand; rest; rest &= rest - 1) {
          const int r = __ffs(rest) - 1;
          uint32_t x = w[0];
#pragma unroll
          for (int q = 1; q < 8; ++q) x = (r & 7) == q ? w[q] : x;
          const uint32_t by = (x >> ((r >> 3) << 3)) & 0xFFu, bit = 1u << r;
          gA |= by > la ? bit : 0u;
          eA |= by == la ? bit : 0u;
          gB |= by > lb ? bit : 0u;
          eB |= by == lb ? bit : 0u;
        }
        zgtA |= zeqA & gA;
        zeqA &= eA;
        zgtB |= zeqB & gB;
        zeqB &= eB & (zeqA | zgtA);
      }
      continue;
    }
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
        } else if (L1Z && A.byte[j] == 0u) {
          // the L1Z variant also covers deeper lo bytes 0x00 (small ranks)
          cmp_block2_z(w, A.lv[j], B.lv[j], gA, eA, gB, eB);
        } else {
          cmp_block2(w, A.lv[j], B.lv[j], gA, eA, gB, eB);
        }
        zgtA |= zeqA & gA;
        zeqA &= eA & ~gA;
        zgtB |= zeqB & gB;
        zeqB &= eB & ~gB & (zeqA | zgtA);
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
    cmp_block2(in.w, A.lv[0], B.lv[0], gA, eA, gB, eB);
  } else {
    cmp_block_vbs(in.w, A.lv[0], gA, eA);
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

// PP-VBS, deep slices in level-2 rank space (BSB_DEEP_RANK2): all deep levels
// share one packed space per block, so the row-space <-> packed conversion
// (one butterfly setup) happens once per block instead of once per level.
template <bool BETWEEN, bool STATS>
__device__ __forceinline__ uint32_t scan_tile_vbs_rank2(const VbsDesc& d, const Leg& A,
                                                        const Leg& B, int64_t tile, int64_t b,
                                                        uint32_t valid, const TileIn& in,
                                                        StatAcc* st, int* depth_out) {
  const int K = d.K;
  uint32_t zeqA = valid, zgtA = 0, eqfA = 0;
  uint32_t zeqB = valid, zgtB = 0, eqfB = 0;
  const int maxlen = BETWEEN ? (A.len > B.len ? A.len : B.len) : A.len;
  int depth = 0;
  vbs_level1<BETWEEN, STATS>(A, B, K, valid, in, zeqA, zgtA, eqfA, zeqB, zgtB, eqfB, st, depth);
  const bool any_deep = BETWEEN ? ((zeqA | zeqB) != 0) : (zeqA != 0);
  if (maxlen >= 2 && __any_sync(kFull, any_deep)) {
    const ExpandNet net = expand_setup(in.m2);
    uint32_t pzA = compress_apply(net, zeqA);
    uint32_t pzB = BETWEEN ? compress_apply(net, zeqB) : 0u;
    // deep rows already known to pass GE(lo) at level 1 (row-space results)
    const uint32_t passA1 = BETWEEN ? compress_apply(net, zgtA | eqfA) : 0u;
    uint32_t pgtA = 0, peqA = 0, pgtB = 0, peqB = 0;
    const int c2 = __popc(in.m2);
    const uint32_t incl = warp_incl_scan((uint32_t)c2);
    const int64_t start = in.base + (int64_t)(incl - c2);
    const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
    const int nwmax = __reduce_max_sync(kFull, any_deep ? ((c2 + 3) >> 2) : 0);
    int rc = c2;  // bytes of the current level (reference accounting)
    for (int j = 2; j <= maxlen; ++j) {
      const bool act = BETWEEN ? ((pzA | pzB) != 0) : (pzA != 0);
      if (!__any_sync(kFull, act)) break;
      Run run;
      load_run(d.deep[j - 1], start, c2, act, run);
      const uint32_t mnext = (j < K && act) ? __ldg(d.exist[j] + b) : 0u;
      uint32_t pgA, peA, pgB, peB;
      if (BETWEEN && A.byte[j - 1] != B.byte[j - 1])
        cmp_run<true>(run, nwmax, A.lv[j - 1], B.lv[j - 1], pgA, peA, pgB, peB);
      else
        cmp_run<false>(run, nwmax, A.lv[j - 1], A.lv[j - 1], pgA, peA, pgB, peB);
      const uint32_t rnext = compress_apply(net, mnext);  // M_{j+1} in packed space
      if (act) {
        depth = j;
        stat_level<STATS>(st, j - 1, rc);
      }
      rc = __popc(rnext);
      vbs_transition(j, A.len, K, pgA & lowm, peA & lowm, rnext, pzA, pgtA, peqA);
      if (BETWEEN) {
        vbs_transition(j, B.len, K, pgB & lowm, peB & lowm, rnext, pzB, pgtB, peqB);
        pzB &= pzA | pgtA | peqA | passA1;
      }
    }
    zgtA |= expand_apply(net, pgtA);
    eqfA |= expand_apply(net, peqA);
    if (BETWEEN) zgtB |= expand_apply(net, pgtB);
  }
  if (STATS) *depth_out = depth;
  if (BETWEEN) return valid & (zgtA | eqfA) & ~zgtB;
  return finalize_op(A.op, zgtA, eqfA, valid);
}

// PP-VBS, deep levels paired into uint16 planes (BSB_DEEP_PLANES), compared
// cooperatively: after the level-1 SWAR pass (lane = block), the warp walks
// the tile's deep rows one per lane (coalesced 2-byte loads, 8 slots in
// flight), compares plane values against the literal planes, resolves ties
// with the deep-row existence bitmap, ballots two flag words per 32 deep rows,
// and each lane finally pulls its block's window of flags and expands it to
// row space with one butterfly.  Requires every literal's last byte to be
// non-zero (dictionary codes always are; the host falls back otherwise).
// VT = uint32_t for columns with at most 2 planes (max_len <= 5), uint64_t else.
template <bool BETWEEN, typename VT>
__device__ __forceinline__ uint32_t scan_tile_vbs_planes(const VbsDesc& d, const Leg& A,
                                                         const Leg& B, int64_t tile, int64_t b,
                                                         uint32_t valid, const TileIn& in) {
  constexpr int G = 12;  // 32-deep-row slots per group: one round trip per plane per group
  constexpr int VB = 8 * (int)sizeof(VT);  // value bits: planes packed big-endian
  const int lane = threadIdx.x & 31;
  const int K = d.K;
  uint32_t zeqA = valid, zgtA = 0, eqfA = 0;
  uint32_t zeqB = valid, zgtB = 0, eqfB = 0;
  int depth = 0;
  vbs_level1<BETWEEN, false>(A, B, K, valid, in, zeqA, zgtA, eqfA, zeqB, zgtB, eqfB, nullptr,
                             depth);
  const int lenA = A.len;
  const int lenB = BETWEEN ? B.len : 0;
  const uint32_t cand = BETWEEN ? (zeqA | zeqB) : zeqA;
  if ((lenA >= 2 || lenB >= 2) && __any_sync(kFull, cand != 0)) {
    const int npA = lenA >> 1, npB = lenB >> 1;  // planes holding literal bytes 2..len
    const int np = npA > npB ? npA : npB;        // 1 or 2 (K <= 5) ... up to 4
    const int c2 = __popc(in.m2);
    const uint32_t incl = warp_incl_scan((uint32_t)c2);
    const uint32_t S = __shfl_sync(kFull, incl, 31);
    const int64_t T0 = in.base;
    // literal planes concatenated: big-endian plane 0 | plane 1 (| plane 2 | plane 3)
    VT LA = 0, LB = 0;
#pragma unroll
    for (int p = 0; p < VB / 16; ++p) {
      const VT a = p < np ? ((A.byte[2 * p + 1] << 8) | A.byte[2 * p + 2]) : 0u;
      const VT bb = p < np ? ((B.byte[2 * p + 1] << 8) | B.byte[2 * p + 2]) : 0u;
      LA |= a << (VB - 16 - 16 * p);
      LB |= bb << (VB - 16 - 16 * p);
    }
    const uint32_t* rexA = (lenA >= 2 && lenA < K) ? d.rexist[lenA] : nullptr;
    const uint32_t* rexB = (BETWEEN && lenB >= 2 && lenB < K) ? d.rexist[lenB] : nullptr;
    const uint16_t* pl0 = reinterpret_cast<const uint16_t*>(d.deep[1]) + T0;
    uint32_t keepP = 0, keepQ = 0;
    const int niter = (int)((S + 31) >> 5);
    for (int g = 0; g < niter; g += G) {
      VT V[G];
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const uint32_t qo = (uint32_t)(g + k) * 32u + lane;
        V[k] = (g + k < niter && qo < S) ? (VT)__ldg(pl0 + qo) << (VB - 16) : (VT)0;
      }
      // further planes only for rows tied so far with a leg that has bytes there
      for (int p = 1; p < np; ++p) {
        const uint16_t* pl = reinterpret_cast<const uint16_t*>(d.deep[p + 1]) + T0;
        const int sh = VB - 16 * p;  // compare the planes loaded so far
        const VT pa = p < npA ? (VT)(LA >> sh) : (VT)~(VT)0;  // ~0: leg has no byte here
        const VT pb = p < npB ? (VT)(LB >> sh) : (VT)~(VT)0;
        bool any = false;
        uint32_t need = 0;
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const VT hv = V[k] >> sh;
          const bool t = (g + k < niter) && (hv == pa || (BETWEEN && hv == pb));
          need |= (uint32_t)t << k;
        }
        any = __any_sync(kFull, need != 0);
        if (!any) break;
#pragma unroll
        for (int k = 0; k < G; ++k)
          if ((need >> k) & 1u)
            V[k] |= (VT)__ldg(pl + (g + k) * 32 + lane) << (VB - 16 - 16 * p);
      }
#pragma unroll
      for (int k = 0; k < G; ++k) {
        if (g + k >= niter) break;
        const uint32_t qo = (uint32_t)(g + k) * 32u + lane;
        const bool inA = qo < S && lenA >= 2, inB = qo < S && lenB >= 2;
        bool gA = inA && V[k] > LA, eA = inA && V[k] == LA;
        bool gB = inB && V[k] > LB, eB = inB && V[k] == LB;
        // tie through a literal's last byte: longer codes are greater (vbs.py:276-280)
        if (rexA != nullptr && __any_sync(kFull, eA)) {
          const uint32_t q = (uint32_t)(T0 + qo);
          const bool has = eA && ((__ldg(rexA + (q >> 5)) >> (q & 31)) & 1u);
          gA |= has;
          eA &= !has;
        }
        if (BETWEEN && rexB != nullptr && __any_sync(kFull, eB)) {
          const uint32_t q = (uint32_t)(T0 + qo);
          const bool has = eB && ((__ldg(rexB + (q >> 5)) >> (q & 31)) & 1u);
          gB |= has;
          eB &= !has;
        }
        const uint32_t wp = __ballot_sync(kFull, BETWEEN ? (gA || eA) : gA);
        const uint32_t wq = __ballot_sync(kFull, BETWEEN ? gB : eA);
        if (lane == g + k) {
          keepP = wp;
          keepQ = wq;
        }
      }
    }
    // this block's deep rows are run bits [incl - c2, incl)
    const uint32_t excl = incl - (uint32_t)c2;
    const int w0 = (int)(excl >> 5), sh = (int)(excl & 31);
    const int w1 = w0 + 1 < 32 ? w0 + 1 : 31;
    const uint32_t p0 = __shfl_sync(kFull, keepP, w0 & 31), p1 = __shfl_sync(kFull, keepP, w1);
    const uint32_t q0 = __shfl_sync(kFull, keepQ, w0 & 31), q1 = __shfl_sync(kFull, keepQ, w1);
    const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
    const uint32_t pP = __funnelshift_r(p0, p1, sh) & lowm;
    const uint32_t pQ = __funnelshift_r(q0, q1, sh) & lowm;
    const ExpandNet net = expand_setup(in.m2);
    const uint32_t eP = expand_apply(net, pP), eQ = expand_apply(net, pQ);
    if (BETWEEN) {
      zgtA |= zeqA & eP;  // deep rows at least lo
      zgtB |= zeqB & eQ;  // deep rows strictly above hi
    } else {
      zgtA |= zeqA & eP;
      eqfA |= zeqA & eQ;
    }
  }
  if (BETWEEN) return valid & (zgtA | eqfA) & ~zgtB;
  return finalize_op(A.op, zgtA, eqfA, valid);
}

// PP-VBS with the deep rows stored as their own ByteSlice-like column
// (BSB_DEEP_SLICED).  Level 1 runs lane = row block as usual.  The tied rows
// of every block (compressed with one butterfly set-up) are OR-ed into
// deep-block candidate words in shared memory; then lane t walks deep block
// t through levels 2..len exactly like Alg. 3 (one 256-bit load and a SWAR
// compare per level, early stop per deep block, transitions with the
// deep-row existence words), and each row block expands its window of the
// deep results back to row space.
constexpr int kTileWarps = 8;  // all scan kernels run 256-thread CTAs

template <bool BETWEEN>
__device__ __forceinline__ uint32_t scan_tile_vbs_sliced(const VbsDesc& d, const Leg& A,
                                                         const Leg& B, int64_t tile, int64_t b,
                                                         uint32_t valid, const TileIn& in) {
  __shared__ uint32_t sh[kTileWarps][5][36];
  const int lane = threadIdx.x & 31;
  const int wq = (threadIdx.x >> 5) & (kTileWarps - 1);
  const int K = d.K;
  uint32_t zeqA = valid, zgtA = 0, eqfA = 0;
  uint32_t zeqB = valid, zgtB = 0, eqfB = 0;
  int depth = 0;
  vbs_level1<BETWEEN, false>(A, B, K, valid, in, zeqA, zgtA, eqfA, zeqB, zgtB, eqfB, nullptr,
                             depth);
  const int lenA = A.len;
  const int lenB = BETWEEN ? B.len : 0;
  const int maxlen = lenA > lenB ? lenA : lenB;
  const uint32_t cand = BETWEEN ? (zeqA | zeqB) : zeqA;
  if (maxlen >= 2 && __any_sync(kFull, cand != 0)) {
    const int c2 = __popc(in.m2);
    const uint32_t incl = warp_incl_scan((uint32_t)c2);
    const uint32_t S = __shfl_sync(kFull, incl, 31);
    const int64_t D0 = in.base;
    const int64_t db0 = D0 >> 5;
    const int off0 = (int)(D0 & 31);
    const int ndt = (off0 + (int)S + 31) >> 5;  // deep blocks this tile touches (<= 33)
    const ExpandNet net = expand_setup(in.m2);
    const uint32_t pA = compress_apply(net, zeqA);
    const uint32_t pB = BETWEEN ? compress_apply(net, zeqB) : 0u;
    uint32_t* cA = sh[wq][0];
    uint32_t* cB = sh[wq][1];
    cA[lane] = 0;
    cB[lane] = 0;
    if (lane < 4) {
      cA[32 + lane] = 0;
      cB[32 + lane] = 0;
    }
    __syncwarp();
    const int o = off0 + (int)(incl - (uint32_t)c2);  // block's first deep row, from db0*32
    const int wi = o >> 5, sb = o & 31;
    const bool spill = sb != 0 && sb + c2 > 32;
    if (pA) {
      atomicOr(&cA[wi], pA << sb);
      if (spill) atomicOr(&cA[wi + 1], pA >> (32 - sb));
    }
    if (BETWEEN && pB) {
      atomicOr(&cB[wi], pB << sb);
      if (spill) atomicOr(&cB[wi + 1], pB >> (32 - sb));
    }
    __syncwarp();
    for (int t0 = 0; t0 < ndt; t0 += 32) {
      const int t = t0 + lane;
      const bool has = t < ndt;
      uint32_t zA = has ? cA[t] : 0u, zB = (BETWEEN && has) ? cB[t] : 0u;
      uint32_t gtA = 0, eqA = 0, gtB = 0, eqB = 0;
      const int64_t dbk = db0 + t;
      for (int j = 2; j <= maxlen; ++j) {
        const bool act = BETWEEN ? ((zA | zB) != 0) : (zA != 0);
        if (!__any_sync(kFull, act)) break;
        uint32_t w[8];
        if (act) {
          ldg256(d.deep[j - 1] + dbk * 32, w);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) w[i] = 0;
        }
        const uint32_t nxt = (j < K && act) ? __ldg(d.rexist[j] + dbk) : 0u;
        uint32_t gA, eA, gB, eB;
        if (BETWEEN && A.byte[j - 1] != B.byte[j - 1]) {
          cmp_block2(w, A.lv[j - 1], B.lv[j - 1], gA, eA, gB, eB);
        } else {
          cmp_block(w, A.lv[j - 1], gA, eA);
          gB = gA;
          eB = eA;
        }
        eA &= ~gA;
        eB &= ~gB;
        vbs_transition(j, lenA, K, gA, eA, nxt, zA, gtA, eqA);
        if (BETWEEN) vbs_transition(j, lenB, K, gB, eB, nxt, zB, gtB, eqB);
      }
      __syncwarp();
      if (has) {
        sh[wq][2][t] = BETWEEN ? (gtA | eqA) : gtA;
        sh[wq][3][t] = BETWEEN ? gtB : eqA;
      }
    }
    if (lane < 4) {
      sh[wq][2][ndt + lane] = 0;  // guard words read by the last windows
      sh[wq][3][ndt + lane] = 0;
    }
    __syncwarp();
    const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
    const uint32_t pP = __funnelshift_r(sh[wq][2][wi], sh[wq][2][wi + 1], sb) & lowm;
    const uint32_t pQ = __funnelshift_r(sh[wq][3][wi], sh[wq][3][wi + 1], sb) & lowm;
    const uint32_t eP = expand_apply(net, pP), eQ = expand_apply(net, pQ);
    if (BETWEEN) {
      zgtA |= zeqA & eP;  // deep rows at least lo
      zgtB |= zeqB & eQ;  // deep rows strictly above hi
    } else {
      zgtA |= zeqA & eP;
      eqfA |= zeqA & eQ;
    }
    __syncwarp();
  }
  if (BETWEEN) return valid & (zgtA | eqfA) & ~zgtB;
  return finalize_op(A.op, zgtA, eqfA, valid);
}

// MODE: -1 = dispatch on d.mode at run time (conjunction kernel), else the
// deep layout fixed at compile time (single-predicate scan kernels):
// 0 packed, 1 rank2, 2 planes (32-bit values), 3 sliced, 4 planes (64-bit).
template <bool BETWEEN, bool STATS, int MODE = -1>
__device__ __forceinline__ uint32_t scan_tile_vbs(const VbsDesc& d, const Leg& A,
                                                  const Leg& B, int64_t tile, int64_t b,
                                                  uint32_t valid, const TileIn& in,
                                                  StatAcc* st, int* depth_out) {
  if (MODE == BSB_DEEP_PLANES)  // PLANES, max_len <= 5
    return scan_tile_vbs_planes<BETWEEN, uint32_t>(d, A, B, tile, b, valid, in);
  if (MODE == 4)  // PLANES, max_len > 5
    return scan_tile_vbs_planes<BETWEEN, uint64_t>(d, A, B, tile, b, valid, in);
  if (MODE == BSB_DEEP_SLICED)
    return scan_tile_vbs_sliced<BETWEEN>(d, A, B, tile, b, valid, in);
  if (MODE < 0 && !STATS && d.mode == BSB_DEEP_PLANES) {
    if (d.K <= 5) return scan_tile_vbs_planes<BETWEEN, uint32_t>(d, A, B, tile, b, valid, in);
    return scan_tile_vbs_planes<BETWEEN, uint64_t>(d, A, B, tile, b, valid, in);
  }
  if (MODE < 0 && !STATS && d.mode == BSB_DEEP_SLICED)
    return scan_tile_vbs_sliced<BETWEEN>(d, A, B, tile, b, valid, in);
  if (MODE == BSB_DEEP_RANK2)
    return scan_tile_vbs_rank2<BETWEEN, STATS>(d, A, B, tile, b, valid, in, st, depth_out);
  if (MODE == BSB_DEEP_PACKED)
    return scan_tile_vbs_packed<BETWEEN, STATS>(d, A, B, tile, b, valid, in, st, depth_out);
  if (d.mode == BSB_DEEP_RANK2)
    return scan_tile_vbs_rank2<BETWEEN, STATS>(d, A, B, tile, b, valid, in, st, depth_out);
  return scan_tile_vbs_packed<BETWEEN, STATS>(d, A, B, tile, b, valid, in, st, depth_out);
}

}  // namespace bsb
