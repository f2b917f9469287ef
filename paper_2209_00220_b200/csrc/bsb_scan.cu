// bsb_scan.cu -- scan kernels (ByteSlice, PP-VBS, fused conjunction) and
// their C-ABI launchers.  Kernel bodies live in bsb_scan_impl.cuh.
#include <cstdlib>
#include <cstring>

#include <map>
#include <mutex>
#include <utility>

#include "bsb_scan_impl.cuh"

namespace bsb {

constexpr int kScanThreads = 256;

struct ScanArgs {
  int64_t n_rows;
  int64_t nb;
  int64_t ntiles;
  BsDesc bs;
  VbsDesc vbs;
  Leg A, B;
  const uint32_t* mask;
  uint32_t* out;
  unsigned long long* count;
  int64_t* stats;
  int8_t* depth;
  int32_t skipped_slot;
  int32_t depth_max;  // STATS: 1 = depth[b] = max(depth[b], d) (second BETWEEN leg)
  // bs_scan_small_kernel: count accumulator | arrivals << 48 of the call's stream (count_slot());
  // the last CTA stores the total into *count, so no memset node precedes
  // the kernel
  unsigned long long* slot;
};

// Count slots of the small-column scan: zero at load time, and the kernel
// that used a slot leaves it zero again, so a call needs no memset.  A slot
// belongs to one (stream, capture) pair for the life of the process: kernels
// of one stream -- or of one branch of one captured graph -- never overlap
// (the scan's epilogue comes after its griddepcontrol.wait), so no two
// kernels ever hold a slot at once.  NULL when the arena is used up (the
// caller then zeroes count with a memset as before).
constexpr int kCountSlots = 1 << 16;
__device__ unsigned long long g_count_slots[kCountSlots];
static unsigned long long* count_slot(cudaStream_t s) {
  static unsigned long long* base = [] {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_count_slots);
    return static_cast<unsigned long long*>(p);
  }();
  if (!base) return nullptr;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long cap = 0;
  if (cudaStreamGetCaptureInfo(s, &st, &cap) != cudaSuccess) return nullptr;
  if (st != cudaStreamCaptureStatusActive) cap = 0;
  static std::mutex mu;
  static std::map<std::pair<unsigned long long, cudaStream_t>, int> slots;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(cap, s);
  auto it = slots.find(key);
  if (it == slots.end()) {
    if ((int)slots.size() >= kCountSlots) return nullptr;
    it = slots.emplace(key, (int)slots.size()).first;
  }
  return base + it->second;
}

template <bool STATS>
__device__ __forceinline__ void flush_stats(const ScanArgs& a, StatAcc& st) {
  if (!STATS) return;
#pragma unroll
  for (int j = 0; j < kMaxLevels; ++j) {
    long long w = st.words[j], by = st.bytes[j];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      w += __shfl_xor_sync(kFull, w, d);
      by += __shfl_xor_sync(kFull, by, d);
    }
    if ((threadIdx.x & 31) == 0) {
      if (w) atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + j), (unsigned long long)w);
      if (by)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + 8 + j),
                  (unsigned long long)by);
    }
  }
  long long s = st.skipped;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(kFull, s, d);
  if ((threadIdx.x & 31) == 0 && s)
    atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + a.skipped_slot),
              (unsigned long long)s);
}

template <int LAYOUT>
__device__ __forceinline__ void fetch_tile(const ScanArgs& a, int64_t tile, int64_t b,
                                           uint32_t valid, TileIn& t) {
  if (LAYOUT == BSB_LAYOUT_BYTESLICE)
    fetch_bs(a.bs, b, valid, t);
  else
    fetch_vbs(a.vbs, tile, b, valid, t);
}

template <bool MASKED>
__device__ __forceinline__ uint32_t mask_raw(const ScanArgs& a, int64_t b) {
  if (!MASKED) return kFull;
  return b < a.nb ? __ldg(a.mask + b) : 0u;
}

__device__ __forceinline__ uint32_t tile_valid(int64_t tile, int64_t b, int64_t n_rows) {
  return ((tile + 1) * kTileRows <= n_rows) ? kFull : tail_valid(b, n_rows);
}

// Persistent grid-stride kernel: one warp per tile, the next tile's level-1
// operands (and two tiles ahead, its input-mask word) are fetched while the
// current tile is scanned.
template <int LAYOUT, bool BETWEEN, bool STATS, bool MASKED>
__global__ void __launch_bounds__(kScanThreads, 1)
    scan_kernel(const __grid_constant__ ScanArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cnt = 0;
  StatAcc st;
  if (STATS) {
#pragma unroll
    for (int j = 0; j < kMaxLevels; ++j) st.words[j] = st.bytes[j] = 0;
    st.skipped = 0;
  }
  int64_t tile = warp;
  uint32_t vN = 0, mraw = kFull;
  TileIn inN;
  if (tile < a.ntiles) {
    const int64_t b0 = tile * 32 + lane;
    vN = tile_valid(tile, b0, a.n_rows) & mask_raw<MASKED>(a, b0);
    fetch_tile<LAYOUT>(a, tile, b0, vN, inN);
    mraw = mask_raw<MASKED>(a, (tile + nwarps) * 32 + lane);
  }
  for (; tile < a.ntiles; tile += nwarps) {
    const int64_t b = tile * 32 + lane;
    const uint32_t valid = vN;
    const TileIn in = inN;
    const int64_t nt = tile + nwarps;
    if (nt < a.ntiles) {
      const int64_t bn = nt * 32 + lane;
      vN = tile_valid(nt, bn, a.n_rows) & mraw;
      fetch_tile<LAYOUT>(a, nt, bn, vN, inN);
      mraw = mask_raw<MASKED>(a, (nt + nwarps) * 32 + lane);
    }
    if (STATS && b < a.nb && valid == 0) st.skipped += 1;
    int depth = 0;
    uint32_t res;
    if (LAYOUT == BSB_LAYOUT_BYTESLICE)
      res = scan_tile_bs<BETWEEN, STATS>(a.bs, a.A, a.B, b, valid, in, &st, &depth);
    else
      res = scan_tile_vbs<BETWEEN, STATS>(a.vbs, a.A, a.B, tile, b, valid, in, &st, &depth);
    if (b < a.nb) {
      a.out[b] = res;
      if (STATS && a.depth != nullptr) {
        if (a.depth_max) {
          const int8_t old = a.depth[b];
          a.depth[b] = (int8_t)(depth > old ? depth : old);
        } else {
          a.depth[b] = (int8_t)depth;
        }
      }
    }
    cnt += __popc(res);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(kFull, cnt, d);
  if (lane == 0 && cnt && a.count) atomicAdd(a.count, cnt);
  flush_stats<STATS>(a, st);
}

// ---------------------------------------------------------------------------
// ByteSlice scan without stats: persistent warps, lane = 32-row block, and a
// two-stage software pipeline per warp.  While tile Y's level-2 sectors are
// compared, tile X (the next one) has had its level-1 compare done and its
// level-2 loads issued, and tile X's successor has its level-1 sectors in
// flight: the dependent level-2 round trip (byteslice.py:92-95: a block
// reads slice 2 only while it has tied rows) overlaps a whole tile of work.
struct BsState {
  uint32_t valid, zgtA, zeqA, zgtB, zeqB;
};

template <bool BETWEEN>
__device__ __forceinline__ void bs_level(const uint32_t (&w)[8], const Leg& A, const Leg& B,
                                         int j, BsState& s) {
  if (BETWEEN) {
    uint32_t gA, eA, gB, eB;
    cmp_block2(w, A.pl[j], B.pl[j], gA, eA, gB, eB);
    s.zgtA |= s.zeqA & gA;
    s.zeqA &= eA & ~gA;
    s.zgtB |= s.zeqB & gB;
    s.zeqB &= eB & ~gB & (s.zeqA | s.zgtA);  // hi-leg ties that already fail GE(lo)
  } else {
    uint32_t g, e;
    cmp_block(w, A.pl[j], g, e);
    s.zgtA |= s.zeqA & g;
    s.zeqA &= e & ~g;
  }
}

template <bool BETWEEN>
__device__ __forceinline__ bool bs_tied(const BsState& s) {
  return BETWEEN ? ((s.zeqA | s.zeqB) != 0) : (s.zeqA != 0);
}

// STATS (ScanStats of one non-BETWEEN leg, stats.py:18-45): per lane, the
// blocks that read level j as packed 16-bit counters (bytes = 32 per read,
// added on flush), blocks skipped by the mask, and the block's depth.
template <bool BETWEEN, bool MASKED, bool STATS = false>
__global__ void __launch_bounds__(kScanThreads, 4) bs_scan_kernel(const __grid_constant__ ScanArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int K = a.bs.K;
  const int64_t stride = a.bs.stride;
  const uint8_t* sl = a.bs.slices;
  unsigned long long cnt = 0;
  uint32_t lv[STATS ? kMaxLevels / 2 : 1] = {0};  // level-read counters, 2 x 16 bit
  uint32_t skipped = 0;
  auto valid_of = [&](int64_t tile, uint32_t mword) -> uint32_t {
    return tile_valid(tile, tile * 32 + lane, a.n_rows) & (MASKED ? mword : kFull);
  };
  auto count_level = [&](int j) {
    if (STATS) lv[j >> 1] += 1u << (16 * (j & 1));
  };
  int64_t tX = warp;
  uint32_t vN = 0, mN = kFull, wN[8];
  if (tX < a.ntiles) {
    if (MASKED) mN = mask_raw<true>(a, tX * 32 + lane);
    vN = valid_of(tX, mN);
    if (vN) ldg256(sl + (tX * 32 + lane) * 32, wN);
    if (MASKED) mN = mask_raw<true>(a, (tX + nwarps) * 32 + lane);
  }
  BsState sY;
  uint32_t w2Y[8];
  int64_t tY = -1;
  int dY = 0;
  for (;;) {
    // ---- stage X: level 1 of tile tX, issue its level-2 loads
    const bool haveX = tX < a.ntiles;
    BsState sX;
    uint32_t w2X[8];
    int dX = 0;
    if (haveX) {
      uint32_t w1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w1[q] = wN[q];
      sX.valid = vN;
      const int64_t tn = tX + nwarps;
      if (tn < a.ntiles) {
        vN = valid_of(tn, mN);
        if (vN) ldg256(sl + (tn * 32 + lane) * 32, wN);
        if (MASKED) mN = mask_raw<true>(a, (tn + nwarps) * 32 + lane);
      }
      sX.zgtA = 0;
      sX.zeqA = sX.valid;
      sX.zgtB = 0;
      sX.zeqB = sX.valid;
      bs_level<BETWEEN>(w1, a.A, a.B, 0, sX);
      if (STATS) {
        if (sX.valid) {
          dX = 1;
          count_level(0);
        } else if (tX * 32 + lane < a.nb) {
          ++skipped;
        }
      }
      if (K >= 2 && bs_tied<BETWEEN>(sX)) {
        ldg256_sparse(sl + stride + (tX * 32 + lane) * 32, w2X);
        if (STATS) {
          dX = 2;
          count_level(1);
        }
      }
    }
    // ---- stage Y: levels 2..K of tile tY, result word
    if (tY >= 0) {
      if (K >= 2 && __any_sync(kFull, bs_tied<BETWEEN>(sY))) {
        if (bs_tied<BETWEEN>(sY)) bs_level<BETWEEN>(w2Y, a.A, a.B, 1, sY);
#pragma unroll
        for (int j = 2; j < kMaxLevels; ++j) {
          if (j >= K) break;
          const bool act = bs_tied<BETWEEN>(sY);
          if (!__any_sync(kFull, act)) break;
          if (act) {
            uint32_t w[8];
            ldg256_sparse(sl + (int64_t)j * stride + (tY * 32 + lane) * 32, w);
            if (STATS) {
              dY = j + 1;
              count_level(j);
            }
            bs_level<BETWEEN>(w, a.A, a.B, j, sY);
          }
        }
      }
      const uint32_t res = BETWEEN ? sY.valid & (sY.zgtA | sY.zeqA) & ~sY.zgtB
                                   : finalize_op(a.A.op, sY.zgtA, sY.zeqA, sY.valid);
      const int64_t b = tY * 32 + lane;
      if (b < a.nb) {
        a.out[b] = res;
        if (STATS && a.depth != nullptr) {
          if (a.depth_max) {
            const int8_t old = a.depth[b];
            a.depth[b] = (int8_t)(dY > old ? dY : old);
          } else {
            a.depth[b] = (int8_t)dY;
          }
        }
      }
      cnt += __popc(res);
    }
    if (!haveX) break;
    tY = tX;
    sY = sX;
    dY = dX;
#pragma unroll
    for (int q = 0; q < 8; ++q) w2Y[q] = w2X[q];
    tX += nwarps;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(kFull, cnt, d);
  if (lane == 0 && cnt && a.count) atomicAdd(a.count, cnt);
  if (STATS) {
#pragma unroll
    for (int j = 0; j < kMaxLevels; ++j) {
      unsigned long long w = (lv[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) w += __shfl_xor_sync(kFull, w, d);
      if (lane == 0 && w) {
        atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + j), w);
        atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + 8 + j), 32ull * w);
      }
    }
    unsigned long long sk = skipped;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sk += __shfl_xor_sync(kFull, sk, d);
    if (lane == 0 && sk)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + a.skipped_slot), sk);
  }
}

// Small columns (every tile fits in one wave of warps, e.g. cfg1's 2^24
// rows): the persistent pipeline above leaves each warp a serial chain of
// ~2 round trips per tile.  Here a warp takes T tiles at once and issues
// every tile's sector of one level before comparing any, so the whole scan
// is K dependent round trips (level j+1 only for blocks with tied rows,
// byteslice.py:92-95).
template <bool BETWEEN, int T>
__global__ void __launch_bounds__(kScanThreads, 4) bs_scan_small_kernel(const __grid_constant__ ScanArgs a) {
  // programmatic dependent launch: wait for the stream's previous grid (a
  // no-op without the launch attribute), then let the next one start its
  // launch while this one runs (it waits in turn before touching memory)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int K = a.bs.K;
  const int64_t stride = a.bs.stride;
  const uint8_t* sl = a.bs.slices;
  BsState st[T];
  uint32_t w[T][8];
#pragma unroll
  for (int u = 0; u < T; ++u) {
    const int64_t tile = warp * T + u;
    st[u].valid = tile < a.ntiles ? tail_valid(tile * 32 + lane, a.n_rows) : 0u;
    if (st[u].valid) ldg256(sl + (tile * 32 + lane) * 32, w[u]);
  }
#pragma unroll
  for (int u = 0; u < T; ++u) {
    st[u].zgtA = 0;
    st[u].zeqA = st[u].valid;
    st[u].zgtB = 0;
    st[u].zeqB = st[u].valid;
    if (st[u].valid) bs_level<BETWEEN>(w[u], a.A, a.B, 0, st[u]);
  }
#pragma unroll 1
  for (int j = 1; j < K; ++j) {
    bool any = false;
#pragma unroll
    for (int u = 0; u < T; ++u) {
      const int64_t tile = warp * T + u;
      if (bs_tied<BETWEEN>(st[u])) {
        ldg256_sparse(sl + (int64_t)j * stride + (tile * 32 + lane) * 32, w[u]);
        any = true;
      }
    }
    if (!__any_sync(kFull, any)) break;
#pragma unroll
    for (int u = 0; u < T; ++u)
      if (bs_tied<BETWEEN>(st[u])) bs_level<BETWEEN>(w[u], a.A, a.B, j, st[u]);
  }
  unsigned long long cnt = 0;
#pragma unroll
  for (int u = 0; u < T; ++u) {
    const int64_t b = (warp * T + u) * 32 + lane;
    const uint32_t res = BETWEEN ? st[u].valid & (st[u].zgtA | st[u].zeqA) & ~st[u].zgtB
                                 : finalize_op(a.A.op, st[u].zgtA, st[u].zeqA, st[u].valid);
    if (b < a.nb) a.out[b] = res;
    cnt += __popc(res);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(kFull, cnt, d);
  if (!a.count) return;
  if (!a.slot) {  // count zeroed by the caller's memset
    if (lane == 0 && cnt) atomicAdd(a.count, cnt);
    return;
  }
  // count without a memset node: one atomicAdd per CTA carries its count (low
  // 48 bits) and its arrival (bit 48 up); the CTA that sees every other
  // arrival stores the total and leaves the slot zero
  __shared__ unsigned long long wcnt[kScanThreads / 32];
  if (lane == 0) wcnt[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c = 0;
#pragma unroll
    for (int q = 0; q < kScanThreads / 32; ++q) c += wcnt[q];
    const unsigned long long old = atomicAdd(a.slot, c + (1ull << 48));
    if ((old >> 48) == gridDim.x - 1) {
      *a.count = (old & ((1ull << 48) - 1)) + c;
      atomicExch(a.slot, 0ull);
    }
  }
}

// ---------------------------------------------------------------------------
// Fused conjunction of NP ByteSlice predicates (engine.py:322-332): one pass
// per tile evaluates every predicate and ANDs the results in registers -- no
// intermediate result words in HBM.  Level-1 sectors of all NP columns are
// staged into shared memory by 1-D TMA bulk copies (cp.async.bulk, one
// elected lane, completion on a per-warp mbarrier), two tiles ahead, so the
// registers hold no prefetched data; deeper levels (tied rows only,
// byteslice.py:92-95) are loaded directly, all predicates' loads of one level
// in flight together.  Every predicate is evaluated on the tile's valid rows
// and the results are AND-ed: the same words as the pipelined chain (the
// chain evaluates predicate i on the rows still alive, and AND is
// idempotent).
constexpr int kConjMax = 4;
struct BsConjArgs {
  int64_t n_rows, nb, ntiles;
  BsDesc c[kConjMax];
  Leg A[kConjMax], B[kConjMax];
  int32_t between[kConjMax];
  const uint32_t* mask;
  uint32_t* out;
  unsigned long long* count;
};

template <bool BETWEEN_ANY>
__device__ __forceinline__ void conj_level(const uint32_t (&w)[8], const BsConjArgs& a, int p,
                                           int j, BsState& s) {
  if (BETWEEN_ANY && a.between[p])
    bs_level<true>(w, a.A[p], a.B[p], j, s);
  else
    bs_level<false>(w, a.A[p], a.B[p], j, s);
}
template <bool BANY>
__device__ __forceinline__ bool conj_tied(const BsConjArgs& a, int p, const BsState& s) {
  return BANY && a.between[p] ? ((s.zeqA | s.zeqB) != 0) : (s.zeqA != 0);
}
template <bool BANY>
__device__ __forceinline__ uint32_t conj_result(const BsConjArgs& a, int p, const BsState& s) {
  return BANY && a.between[p] ? s.valid & (s.zgtA | s.zeqA) & ~s.zgtB
                              : finalize_op(a.A[p].op, s.zgtA, s.zeqA, s.valid);
}

// Two-stage pipeline per warp as in bs_scan_kernel: tile X's level-1
// sectors come from the TMA-filled stage and its level-2 loads are issued;
// tile Y (the previous one) consumes its level-2 sectors, runs any deeper
// level, ANDs the NP results and writes the word.
// BANY false: no predicate of the group is a BETWEEN (the second leg's state
// and compares drop out at compile time).
template <int NP, bool MASKED, bool BANY>
__global__ void __launch_bounds__(kScanThreads, 3) bs_conj_kernel(const __grid_constant__ BsConjArgs a) {
  constexpr int kW = kScanThreads / 32;
  __shared__ __align__(128) uint8_t sbuf[kW][2][NP][1024];
  __shared__ __align__(8) uint64_t sbar[kW][2];
  const int lane = threadIdx.x & 31;
  const int wq = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t* bar = sbar[wq];
  auto issue = [&](int st, int64_t tile) {
    if (lane == 0 && tile < a.ntiles) {
      mbar_expect_tx(&bar[st], NP * 1024u);
#pragma unroll
      for (int p = 0; p < NP; ++p)
        bulk_g2s(sbuf[wq][st][p], a.c[p].slices + tile * 1024, 1024u, &bar[st]);
    }
  };
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  issue(0, warp);
  issue(1, warp + nwarps);
  uint32_t phases = 0u;  // bit st = parity to wait for on stage st
  unsigned long long cnt = 0;
  int st = 0;
  BsState sY[NP];
  uint32_t w2Y[NP][8];
  int64_t tY = -1;
  for (int64_t tX = warp;; tX += nwarps) {
    const bool haveX = tX < a.ntiles;
    BsState sX[NP];
    uint32_t w2X[NP][8];
    if (haveX) {
      const int64_t b = tX * 32 + lane;
      uint32_t valid = tile_valid(tX, b, a.n_rows);
      if (MASKED) valid &= b < a.nb ? __ldg(a.mask + b) : 0u;
      mbar_wait(&bar[st], (phases >> st) & 1u);
      phases ^= 1u << st;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const uint4* src = reinterpret_cast<const uint4*>(sbuf[wq][st][p] + lane * 32);
        const uint4 x = src[0], y = src[1];
        const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
        sX[p].valid = valid;
        sX[p].zgtA = 0;
        sX[p].zeqA = valid;
        sX[p].zgtB = 0;
        sX[p].zeqB = BANY ? valid : 0u;
        conj_level<BANY>(w, a, p, 0, sX[p]);
      }
      __syncwarp();  // every lane has read this stage: refill it two tiles ahead
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(st, tX + 2 * nwarps);
      st ^= 1;
#pragma unroll
      for (int p = 0; p < NP; ++p)
        if (a.c[p].K >= 2 && conj_tied<BANY>(a, p, sX[p]))
          ldg256_sparse(a.c[p].slices + a.c[p].stride + b * 32, w2X[p]);
    }
    if (tY >= 0) {
      const int64_t b = tY * 32 + lane;
#pragma unroll
      for (int p = 0; p < NP; ++p)
        if (a.c[p].K >= 2 && conj_tied<BANY>(a, p, sY[p])) conj_level<BANY>(w2Y[p], a, p, 1, sY[p]);
#pragma unroll
      for (int j = 2; j < kMaxLevels; ++j) {
        bool act[NP];
        bool any = false;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          act[p] = j < a.c[p].K && conj_tied<BANY>(a, p, sY[p]);
          any |= act[p];
        }
        if (!__any_sync(kFull, any)) break;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (!act[p]) continue;
          uint32_t w[8];
          ldg256_sparse(a.c[p].slices + (int64_t)j * a.c[p].stride + b * 32, w);
          conj_level<BANY>(w, a, p, j, sY[p]);
        }
      }
      uint32_t res = sY[0].valid;
#pragma unroll
      for (int p = 0; p < NP; ++p) res &= conj_result<BANY>(a, p, sY[p]);
      if (b < a.nb) a.out[b] = res;
      cnt += __popc(res);
    }
    if (!haveX) break;
    tY = tX;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      sY[p] = sX[p];
#pragma unroll
      for (int q = 0; q < 8; ++q) w2Y[p][q] = w2X[p][q];
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(kFull, cnt, d);
  if (lane == 0 && cnt) atomicAdd(a.count, cnt);
}

// Trivial predicates (vbs.py:200-208): true -> mask & valid, false -> 0.
__global__ void trivial_kernel(int64_t n_rows, int64_t nb, const uint32_t* mask, int value,
                               uint32_t* out, unsigned long long* count) {
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
  if ((threadIdx.x & 31) == 0 && c && count) atomicAdd(count, c);
}

// ------------------------------------------------------------ host helpers

static void fill_leg(Leg& L, int op, uint64_t code, int len, int levels) {
  std::memset(&L, 0, sizeof(L));
  L.op = op;
  L.len = len;
  for (int j = 0; j <= kMaxLevels; ++j) {
    uint32_t byte = 0;
    if (j < levels) byte = (uint32_t)((code >> (8 * (levels - 1 - j))) & 0xFF);
    L.byte[j] = byte;
    if (j < kMaxLevels) {
      L.lv[j] = make_level_lit(byte);
      L.pl[j] = make_plane_lit(byte);
    }
  }
}

// ByteSlice literal: left-aligned like the codes, pred.length ignored
// (byteslice.py:81).
static void bs_leg(Leg& L, int op, uint64_t code, int width_bits, int K) {
  const int shift = 8 * K - width_bits;
  const uint64_t aligned = shift >= 64 ? 0 : (code << shift);
  fill_leg(L, op, aligned, K, K);
}

static bool pred_ok(const bsb_pred* p) {
  if (!p) return false;
  if (p->trivial >= 0) return true;
  return p->op >= BSB_EQ && p->op <= BSB_BETWEEN;
}

template <typename KernelT>
static int launch_scan(KernelT kern, const ScanArgs& a, cudaStream_t s) {
  const int grid = persistent_grid(kern, kScanThreads, kScanThreads / 32, a.ntiles);
  kern<<<grid, kScanThreads, 0, s>>>(a);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

static int run_trivial(int64_t n, const bsb_pred* p, const uint32_t* mask, uint32_t* out,
                       uint64_t* count, int64_t* stats, int8_t* depth, int levels,
                       cudaStream_t s) {
  const int64_t nb = (n + 31) / 32;
  if (count) BSB_CUDA(cudaMemsetAsync(count, 0, sizeof(uint64_t), s));
  int grid = (int)((nb + 255) / 256);
  if (grid > 4096) grid = 4096;
  if (grid < 1) grid = 1;
  trivial_kernel<<<grid, 256, 0, s>>>(n, nb, mask, p->trivial, out,
                                      reinterpret_cast<unsigned long long*>(count));
  BSB_LAUNCH_CHECK();
  if (stats) {
    int64_t h[BSB_STATS_WORDS] = {0};
    h[16] = nb;
    h[17] = nb;  // every block counts as skipped (vbs.py:203-204)
    h[18] = levels;
    h[19] = nb;
    BSB_CUDA(cudaMemcpyAsync(stats, h, sizeof(h), cudaMemcpyHostToDevice, s));
    BSB_CUDA(cudaStreamSynchronize(s));  // h is a stack buffer
  }
  if (depth) BSB_CUDA(cudaMemsetAsync(depth, 0, nb, s));
  return BSB_OK;
}

static int g_scan_nomemset = 0;  // bsb_tune("scan_nomemset"): diagnostics (count not zeroed)
void set_scan_nomemset(int64_t v) { g_scan_nomemset = v > 0 ? 1 : 0; }

// Launch with programmatic stream serialization (PDL): the kernel may begin
// launching while the stream's previous kernel runs; it executes
// griddepcontrol.wait before any memory access.  bsb_tune("pdl", 0): plain.
static int g_pdl = -1;
void set_pdl(int64_t v) { g_pdl = v < 0 ? -1 : (v ? 1 : 0); }
static bool pdl_on() {
  if (g_pdl < 0) {
    const char* e = std::getenv("BSB_PDL");
    g_pdl = e ? (std::atoi(e) != 0) : 1;
  }
  return g_pdl != 0;
}
template <typename Kern>
static int launch_pdl(Kern kern, int grid, int block, cudaStream_t s, const ScanArgs& a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BSB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

// Small-column ByteSlice path (bs_scan_small_kernel): when every tile fits
// one wave of 4-tile warps at 4 CTAs per SM; bsb_tune("bs_small", 0) off.
static int g_bs_small = -1;
void set_bs_small(int64_t v) { g_bs_small = v < 0 ? -1 : (v ? 1 : 0); }
static bool small_bs_ok(int64_t ntiles) {
  if (g_bs_small < 0) {
    const char* e = std::getenv("BSB_BS_SMALL");
    g_bs_small = e ? (std::atoi(e) != 0) : 1;
  }
  return g_bs_small && ntiles <= (int64_t)sm_count() * 4 * (kScanThreads / 32) * 4;
}

template <int LAYOUT>
static int scan_dispatch(ScanArgs& a, const bsb_pred* p, int levels, cudaStream_t s) {
  const bool between = p->op == BSB_BETWEEN;
  const bool stats = a.stats != nullptr;
  const bool small = !stats && LAYOUT == BSB_LAYOUT_BYTESLICE && !a.mask && small_bs_ok(a.ntiles);
  if (small && a.count) a.slot = count_slot(s);
  if (a.count && !a.slot && !g_scan_nomemset)
    BSB_CUDA(cudaMemsetAsync(a.count, 0, sizeof(uint64_t), s));
  if (!stats) {
    if (LAYOUT == BSB_LAYOUT_BYTESLICE) {
      if (small) {
        constexpr int T = 4;
        const int64_t warps = (a.ntiles + T - 1) / T;
        const int grid = (int)((warps + kScanThreads / 32 - 1) / (kScanThreads / 32));
        return launch_pdl(between ? bs_scan_small_kernel<true, T> : bs_scan_small_kernel<false, T>,
                          grid, kScanThreads, s, a);
      }
      if (a.mask) {
        if (between) return launch_scan(bs_scan_kernel<true, true>, a, s);
        return launch_scan(bs_scan_kernel<false, true>, a, s);
      }
      if (between) return launch_scan(bs_scan_kernel<true, false>, a, s);
      return launch_scan(bs_scan_kernel<false, false>, a, s);
    }
    if (a.mask) {
      if (between) return launch_scan(scan_kernel<LAYOUT, true, false, true>, a, s);
      return launch_scan(scan_kernel<LAYOUT, false, false, true>, a, s);
    }
    if (between) return launch_scan(scan_kernel<LAYOUT, true, false, false>, a, s);
    return launch_scan(scan_kernel<LAYOUT, false, false, false>, a, s);
  }
  // Stats path: reproduce the reference's two pipelined legs exactly
  // (vbs.py:299-304, stats.py:47-67).
  int64_t h[BSB_STATS_WORDS] = {0};
  h[16] = a.nb;
  h[18] = levels;
  BSB_CUDA(cudaMemcpyAsync(a.stats, h, sizeof(h), cudaMemcpyHostToDevice, s));
  // one non-BETWEEN leg with stats: ByteSlice through the pipelined kernel
  // (per-lane 16-bit level counters: at most 65535 tiles per warp)
  auto leg = [&](const ScanArgs& g) -> int {
    if (LAYOUT == BSB_LAYOUT_BYTESLICE) {
      auto k = g.mask ? bs_scan_kernel<false, true, true> : bs_scan_kernel<false, false, true>;
      const int grid = persistent_grid(k, kScanThreads, kScanThreads / 32, g.ntiles);
      const int64_t per_warp = (g.ntiles + (int64_t)grid * 8 - 1) / ((int64_t)grid * 8);
      if (per_warp < 65536) {
        k<<<grid, kScanThreads, 0, s>>>(g);
        BSB_LAUNCH_CHECK();
        return BSB_OK;
      }
    }
    return g.mask ? launch_scan(scan_kernel<LAYOUT, false, true, true>, g, s)
                  : launch_scan(scan_kernel<LAYOUT, false, true, false>, g, s);
  };
  if (!between) {
    a.skipped_slot = 17;
    a.depth_max = 0;
    return leg(a);
  }
  uint32_t* tmp = nullptr;
  BSB_CUDA(cudaMallocAsync(&tmp, (size_t)a.nb * 4 + 4, s));
  ScanArgs leg1 = a;
  leg1.B = a.B;
  leg1.out = tmp;
  leg1.skipped_slot = 17;
  leg1.depth_max = 0;
  // leg 1: GE(lo) over the caller's mask; leg 2: LE(hi) over leg 1's result
  leg1.A.op = BSB_GE;
  unsigned long long* dummy = nullptr;
  BSB_CUDA(cudaMallocAsync(&dummy, 8, s));
  BSB_CUDA(cudaMemsetAsync(dummy, 0, 8, s));
  leg1.count = dummy;
  int rc = leg(leg1);
  if (rc) return rc;
  ScanArgs leg2 = a;
  leg2.A = a.B;
  leg2.A.op = BSB_LE;
  leg2.mask = tmp;
  leg2.skipped_slot = 19;
  leg2.depth_max = 1;
  rc = leg(leg2);
  if (rc) return rc;
  BSB_CUDA(cudaFreeAsync(tmp, s));
  BSB_CUDA(cudaFreeAsync(dummy, s));
  return BSB_OK;
}

}  // namespace bsb

using namespace bsb;

extern "C" int bsb_byteslice_scan(const bsb_byteslice* col, const bsb_pred* pred,
                                  const uint32_t* mask, uint32_t* out_words, uint64_t* count,
                                  int64_t* stats, int8_t* depth, void* stream) {
  if (!col || !pred_ok(pred) || !out_words || (!count && stats) || col->n_rows <= 0)
    return BSB_EINVAL;
  if (col->n_slices < 1 || col->n_slices > kMaxLevels) return BSB_ERANGE;
  cudaStream_t s = as_stream(stream);
  if (pred->trivial >= 0)
    return run_trivial(col->n_rows, pred, mask, out_words, count, stats, depth, col->n_slices,
                       s);
  ScanArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_rows = col->n_rows;
  a.nb = (col->n_rows + 31) / 32;
  a.ntiles = (a.nb + 31) / 32;
  a.bs.slices = col->slices;
  a.bs.stride = col->stride;
  a.bs.K = col->n_slices;
  const int K = col->n_slices;
  if (pred->op == BSB_BETWEEN) {
    bs_leg(a.A, BSB_GE, pred->code, col->width_bits, K);
    bs_leg(a.B, BSB_LE, pred->code2, col->width_bits, K);
  } else {
    bs_leg(a.A, pred->op, pred->code, col->width_bits, K);
    a.B = a.A;
  }
  a.mask = mask;
  a.out = out_words;
  a.count = reinterpret_cast<unsigned long long*>(count);
  a.stats = stats;
  a.depth = depth;
  return scan_dispatch<BSB_LAYOUT_BYTESLICE>(a, pred, K, s);
}

static void fill_vbs_desc(VbsDesc& d, const bsb_vbs* col) {
  std::memset(&d, 0, sizeof(d));
  d.bs1 = col->bs1;
  d.K = col->max_len;
  d.mode = col->deep_mode;
  for (int j = 0; j < kMaxLevels; ++j) {
    d.deep[j] = col->deep[j];
    d.exist[j] = col->exist[j];
    d.dir[j] = col->block_dir[j];
    d.rexist[j] = col->rexist[j];
  }
}

namespace bsb {
int vbs_rows_scan(const VbsDesc& d, int64_t n_rows, const bsb_pred* p, const uint32_t* mask,
                  uint32_t* out, uint64_t* count, int64_t* stats, int8_t* depth,
                  cudaStream_t s);
int vbs_sliced_scan(const VbsDesc& d, int64_t n_rows, int64_t deep_rows, const Leg& A,
                    const Leg& B, bool between,
                    const uint32_t* mask, uint32_t* out, unsigned long long* count,
                    cudaStream_t s);
int vbs_ds_scan(const VbsDesc& d, int64_t n_rows, int64_t stride, int64_t deep_rows,
                int deep1_shared, const Leg& A, const Leg& B, bool between,
                const uint32_t* mask, uint32_t* out, unsigned long long* count,
                cudaStream_t s, const unsigned long long* gate = nullptr,
                unsigned long long gate_max = 0);
void shallow_thresholds(const Leg& A, const Leg& B, bool between, int& tP, int& tQ,
                        uint32_t& inv);
int vbs_ds_stats_scan(const VbsDesc& d, int64_t n_rows, int64_t stride, int deep1_shared,
                      const Leg& A, const Leg& B, bool between, int tP, int tQ, uint32_t inv,
                      const uint32_t* mask, uint32_t* out, unsigned long long* count,
                      int64_t* stats, int8_t* depth, cudaStream_t s);
}

namespace bsb {
bool ds_enabled(bool masked);  // bsb_tune("ds_enable") / BSB_DS
bool ds_zonemap_enabled();     // bsb_tune("ds_zonemap") / BSB_DS_ZONEMAP
}

// Mask density (masked-in rows per column row) at or below which a masked
// SLICED scan runs the compacted kernel (work over the masked-in blocks
// only); above it the column is scanned whole and the mask AND-ed into the
// result words (EPI), which is cheaper for dense masks (cfg5 segment, z1:
// 0.75 % 119 vs 215 us, 5 % 211 vs 215, 20 % 252 vs 215).
static double g_sparse_frac = -1.0;
static double sparse_frac() {
  if (g_sparse_frac < 0) {
    const char* e = std::getenv("BSB_SPARSE_FRAC");
    g_sparse_frac = e ? std::atof(e) : 0.06;
  }
  return g_sparse_frac;
}

// Row count of a mask estimated from 8192 evenly spaced words (the gate of a
// masked scan called outside a conjunction chain: a heuristic only -- both
// gated kernels return the same words).
__global__ void mask_sample_kernel(const uint32_t* __restrict__ mask, int64_t nb,
                                   unsigned long long* est) {
  constexpr int64_t kSample = 8192;
  const int64_t step = nb > kSample ? nb / kSample : 1;
  const int64_t n = nb > kSample ? kSample : nb;
  unsigned long long c = 0;
#pragma unroll 8
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) c += __popc(__ldg(mask + i * step));
  for (int dd = 16; dd > 0; dd >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, dd);
  __shared__ unsigned long long tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&tot, c);
  __syncthreads();
  if (threadIdx.x == 0) *est = tot * (unsigned long long)step;
}
namespace bsb {
void set_sparse_ppm(int64_t ppm) { g_sparse_frac = ppm < 0 ? -1.0 : (double)ppm * 1e-6; }  // < 0: default
}

// Fused ByteSlice pair of a conjunction chain (bs_conj_kernel); mask may be
// NULL.  count is zeroed here.
static int bs_conj2(const bsb_byteslice* c0, const bsb_pred* p0, const bsb_byteslice* c1,
                    const bsb_pred* p1, const uint32_t* mask, uint32_t* out, uint64_t* count,
                    cudaStream_t s) {
  BsConjArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_rows = c0->n_rows;
  a.nb = (a.n_rows + 31) / 32;
  a.ntiles = (a.nb + 31) / 32;
  const bsb_byteslice* cs[2] = {c0, c1};
  const bsb_pred* ps[2] = {p0, p1};
  for (int p = 0; p < 2; ++p) {
    const int K = cs[p]->n_slices;
    a.c[p].slices = cs[p]->slices;
    a.c[p].stride = cs[p]->stride;
    a.c[p].K = K;
    a.between[p] = ps[p]->op == BSB_BETWEEN;
    if (a.between[p]) {
      bs_leg(a.A[p], BSB_GE, ps[p]->code, cs[p]->width_bits, K);
      bs_leg(a.B[p], BSB_LE, ps[p]->code2, cs[p]->width_bits, K);
    } else {
      bs_leg(a.A[p], ps[p]->op, ps[p]->code, cs[p]->width_bits, K);
      a.B[p] = a.A[p];
    }
  }
  a.mask = mask;
  a.out = out;
  a.count = reinterpret_cast<unsigned long long*>(count);
  BSB_CUDA(cudaMemsetAsync(count, 0, sizeof(uint64_t), s));
  const bool bany = a.between[0] || a.between[1];
  auto go = [&](auto kern) -> int {
    static bool carved[4] = {false, false, false, false};
    const int ki = (mask != nullptr) + 2 * bany;
    if (!carved[ki]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      carved[ki] = true;
    }
    const int grid = persistent_grid(kern, kScanThreads, kScanThreads / 32, a.ntiles);
    kern<<<grid, kScanThreads, 0, s>>>(a);
    BSB_LAUNCH_CHECK();
    return BSB_OK;
  };
  if (bany) return mask ? go(bs_conj_kernel<2, true, true>) : go(bs_conj_kernel<2, false, true>);
  return mask ? go(bs_conj_kernel<2, true, false>) : go(bs_conj_kernel<2, false, false>);
}

static int g_stats_rows = 0;  // bsb_tune("stats_rows"): PP-VBS stats via the row kernel
static bool stats_rows() { return g_stats_rows != 0; }
namespace bsb {
void set_stats_rows(int64_t v) { g_stats_rows = v > 0 ? 1 : 0; }  // < 0: default (off)
}

static int g_fuse_bs = -1;  // bsb_tune("conj_fuse") / BSB_CONJ_FUSE: fused ByteSlice pairs
static bool fuse_bs() {
  if (g_fuse_bs < 0) {
    const char* e = std::getenv("BSB_CONJ_FUSE");
    g_fuse_bs = e ? std::atoi(e) : 1;
  }
  return g_fuse_bs != 0;
}
namespace bsb {
void set_conj_fuse(int64_t v) { g_fuse_bs = v < 0 ? -1 : (v ? 1 : 0); }  // < 0: default
}

// gate_count (conjunction chains, masked SLICED scans): device count of the
// input mask's rows; the compacted deep-space kernel runs when it is <=
// sparse_frac * n_rows, the EPI one otherwise (both launched, one exits).
static int vbs_scan_impl(const bsb_vbs* col, const bsb_pred* pred, const uint32_t* mask,
                         uint32_t* out_words, uint64_t* count, int64_t* stats, int8_t* depth,
                         cudaStream_t s, const unsigned long long* gate_count) {
  if (!col || !pred_ok(pred) || !out_words || !count || col->n_rows <= 0) return BSB_EINVAL;
  if (col->max_len < 1 || col->max_len > kMaxLevels) return BSB_ERANGE;
  const int K = col->max_len;
  if (pred->trivial >= 0)
    return run_trivial(col->n_rows, pred, mask, out_words, count, stats, depth, K, s);
  ScanArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_rows = col->n_rows;
  a.nb = (col->n_rows + 31) / 32;
  a.ntiles = (a.nb + 31) / 32;
  fill_vbs_desc(a.vbs, col);
  auto bad_len = [&](int l) { return l < 1 || l > K; };
  if (pred->op == BSB_BETWEEN) {
    if (bad_len(pred->length) || bad_len(pred->length2)) return BSB_ERANGE;
    fill_leg(a.A, BSB_GE, pred->code, pred->length, pred->length);
    fill_leg(a.B, BSB_LE, pred->code2, pred->length2, pred->length2);
  } else {
    if (bad_len(pred->length)) return BSB_ERANGE;
    fill_leg(a.A, pred->op, pred->code, pred->length, pred->length);
    a.B = a.A;
  }
  a.mask = mask;
  a.out = out_words;
  a.count = reinterpret_cast<unsigned long long*>(count);
  a.stats = stats;
  a.depth = depth;
  if (col->deep_mode == BSB_DEEP_SLICED && stats != nullptr) {
    // ScanStats: the deep-space kernel with survival counters when the column
    // has what it needs, else the row-parallel kernel (bsb_tune stats_rows=1
    // forces the latter)
    if (K >= 2 && !stats_rows() &&
        (col->deep[0] || (col->deep1_shared > 0 && bsb::ds_zonemap_enabled()))) {
      int tP, tQ;
      uint32_t inv;
      const bool between = pred->op == BSB_BETWEEN;
      shallow_thresholds(a.A, a.B, between, tP, tQ, inv);
      return vbs_ds_stats_scan(a.vbs, a.n_rows, col->stride,
                               col->deep[0] ? 0 : col->deep1_shared, a.A, a.B, between, tP, tQ,
                               inv, mask, out_words, a.count, stats, depth, s);
    }
    return vbs_rows_scan(a.vbs, a.n_rows, pred, mask, out_words, count, stats, depth, s);
  }
  switch (col->deep_mode) {
    case BSB_DEEP_PACKED: return scan_dispatch<BSB_LAYOUT_PPVBS>(a, pred, K, s);
    case BSB_DEEP_SLICED:
      if (K >= 2 && bsb::ds_enabled(mask != nullptr) &&
          (col->deep[0] || (col->deep1_shared > 0 && bsb::ds_zonemap_enabled()))) {
        if (mask) {
          // gate: the chain's running count, else a sampled estimate
          const unsigned long long gmax =
              (unsigned long long)(sparse_frac() * (double)col->n_rows);
          unsigned long long* est = nullptr;
          if (!gate_count && gmax > 0) {
            BSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&est), 8, s));
            mask_sample_kernel<<<1, 1024, 0, s>>>(mask, a.nb, est);
            BSB_LAUNCH_CHECK();
          }
          BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
          const int rc = vbs_ds_scan(a.vbs, a.n_rows, col->stride, col->deep_len[1],
                                     col->deep1_shared, a.A, a.B, pred->op == BSB_BETWEEN,
                                     mask, out_words, a.count, s,
                                     gate_count ? gate_count : est, gmax);
          if (est) BSB_CUDA(cudaFreeAsync(est, s));
          return rc;
        }
        return vbs_ds_scan(a.vbs, a.n_rows, col->stride, col->deep_len[1], col->deep1_shared,
                           a.A, a.B, pred->op == BSB_BETWEEN, mask, out_words, a.count, s);
      }
      return vbs_sliced_scan(a.vbs, a.n_rows, K >= 2 ? col->deep_len[1] : 0, a.A, a.B,
                             pred->op == BSB_BETWEEN, mask, out_words, a.count, s);
    default: return BSB_EINVAL;
  }
}

extern "C" int bsb_vbs_scan(const bsb_vbs* col, const bsb_pred* pred, const uint32_t* mask,
                            uint32_t* out_words, uint64_t* count, int64_t* stats, int8_t* depth,
                            void* stream) {
  return vbs_scan_impl(col, pred, mask, out_words, count, stats, depth, as_stream(stream),
                       nullptr);
}

// ------------------------------------------------------------- conjunction
// engine.py:322-332: each predicate's scan takes the running result as its
// input mask.  Run as a chain of the per-layout scan kernels (each with its
// own prefetch pipeline; a block whose mask word is 0 loads no slice bytes),
// alternating two result buffers.  Measured faster than a single fused
// kernel that serialises every predicate's loads per tile (cfg4: 211 vs
// 334 us; cfg5 shard: 1.32 vs 1.94 ms).
extern "C" int bsb_conj_scan(int32_t k, const bsb_column_ref* cols, const bsb_pred* preds,
                             const uint32_t* mask, uint32_t* out_words, uint64_t* count,
                             void* stream) {
  if (k < 0 || k > BSB_MAX_CONJ || (k > 0 && (!cols || !preds)) || !out_words || !count)
    return BSB_EINVAL;
  cudaStream_t s = as_stream(stream);
  int64_t n = -1;
  bool all_false = false;
  int live[BSB_MAX_CONJ];
  int m = 0;
  for (int i = 0; i < k; ++i) {
    const bsb_column_ref& c = cols[i];
    const bsb_pred* p = &preds[i];
    if (!pred_ok(p)) return BSB_EINVAL;
    int64_t ni;
    if (c.layout == BSB_LAYOUT_BYTESLICE) {
      if (!c.byteslice) return BSB_EINVAL;
      ni = c.byteslice->n_rows;
    } else if (c.layout == BSB_LAYOUT_PPVBS) {
      if (!c.vbs) return BSB_EINVAL;
      ni = c.vbs->n_rows;
      const int K = c.vbs->max_len;
      auto bad = [&](int l) { return l < 1 || l > K; };
      if (p->trivial < 0 && (bad(p->length) || (p->op == BSB_BETWEEN && bad(p->length2))))
        return BSB_ERANGE;
    } else {
      return BSB_EINVAL;
    }
    if (n >= 0 && ni != n) return BSB_EINVAL;
    n = ni;
    if (p->trivial == 0) all_false = true;
    if (p->trivial >= 0) continue;  // constant true: no-op in a conjunction
    live[m++] = i;
  }
  if (n < 0) return BSB_EINVAL;  // need at least one column to know n_rows
  if (all_false || m == 0) {
    bsb_pred f;
    std::memset(&f, 0, sizeof(f));
    f.trivial = all_false ? 0 : 1;
    return run_trivial(n, &f, mask, out_words, count, nullptr, nullptr, 0, s);
  }
  const int64_t nb = (n + 31) / 32;
  uint32_t* tmp = nullptr;
  // tmp words + one slot holding the running mask's row count for the
  // sparse-mask gate of masked PP-VBS scans
  if (m > 1) BSB_CUDA(cudaMallocAsync(&tmp, (size_t)nb * 4 + 64, s));
  unsigned long long* gate =
      m > 1 ? reinterpret_cast<unsigned long long*>(
                  reinterpret_cast<uintptr_t>(tmp + nb + 8) & ~uintptr_t(7))
            : nullptr;
  // steps: consecutive ByteSlice predicates run as fused pairs (one kernel,
  // AND in registers), everything else one scan each
  int step_first[BSB_MAX_CONJ], step_len[BSB_MAX_CONJ], nsteps = 0;
  for (int t = 0; t < m;) {
    const bool pair = fuse_bs() && t + 1 < m &&
                      cols[live[t]].layout == BSB_LAYOUT_BYTESLICE &&
                      cols[live[t + 1]].layout == BSB_LAYOUT_BYTESLICE;
    step_first[nsteps] = t;
    step_len[nsteps++] = pair ? 2 : 1;
    t += pair ? 2 : 1;
  }
  const uint32_t* running = mask;
  for (int k2 = 0; k2 < nsteps; ++k2) {
    const int t = step_first[k2];
    const int i = live[t];
    // the last step writes out_words; earlier ones alternate through tmp/out
    uint32_t* dst = ((nsteps - 1 - k2) % 2 == 0) ? out_words : tmp;
    int rc;
    if (step_len[k2] == 2) {
      const int i2 = live[t + 1];
      rc = bs_conj2(cols[i].byteslice, &preds[i], cols[i2].byteslice, &preds[i2], running, dst,
                    count, s);
    } else if (cols[i].layout == BSB_LAYOUT_BYTESLICE) {
      rc = bsb_byteslice_scan(cols[i].byteslice, &preds[i], running, dst, count, nullptr,
                              nullptr, s);
    } else {
      const bool gated = k2 > 0;  // running = the previous step's words, count = its rows
      if (gated) BSB_CUDA(cudaMemcpyAsync(gate, count, 8, cudaMemcpyDeviceToDevice, s));
      rc = vbs_scan_impl(cols[i].vbs, &preds[i], running, dst, count, nullptr, nullptr, s,
                         gated ? gate : nullptr);
    }
    if (rc) {
      if (tmp) cudaFreeAsync(tmp, s);
      return rc;
    }
    running = dst;
  }
  if (tmp) BSB_CUDA(cudaFreeAsync(tmp, s));
  return BSB_OK;
}
