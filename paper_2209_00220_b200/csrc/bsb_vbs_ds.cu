// bsb_vbs_ds.cu -- PP-VBS scan in deep-row space (SLICED layout with the
// deep rows' first byte, deep[0]).
//
// The reference's Alg. 3 (vbs.py:222-289) classifies each row by its own
// bytes only, so the rows split cleanly by code length:
//   * a row with a 1-byte code ("shallow", M_2 bit 0) is decided at level 1:
//     gt = byte > lit, eq_final = byte == lit only when the literal has one
//     byte (a shorter code tied on its own bytes is less, vbs.py:273-275);
//   * a row with a longer code ("deep") runs levels 1..len entirely on the
//     deep-row ByteSlice column: level-1 byte from deep[0], byte j from
//     deep[j-1], existence of byte j+1 from rexist[j] (byte 2 always exists).
// Row space therefore needs no level-1 tie masks and no pext into deep-row
// order: phase 1 (lane = row block) computes the shallow rows' result and the
// block's deep-row offset; phase 2 (lane = deep block of the super-tile) runs
// Alg. 3 over the deep rows with early stop per deep block and writes one
// final-result word per deep block; phase 3 deposits each row block's window
// of deep results at its M_2 lanes (pdep) and writes the result word.
//
// L1 = false: the shallow rows cannot match (a BETWEEN whose legs share their
// first byte with a multi-byte lo literal, or EQ with a multi-byte literal),
// so phase 1 reads only the M_2 words -- no first-slice bytes at all.
// Unmasked scans only; masked scans (conjunction chains) use the SLICED
// kernel, which skips the loads of masked-out blocks.
#include <cstdlib>
#include <cstring>

#include "bsb_scan_impl.cuh"

namespace bsb {

constexpr int kDsThreads = 256;
constexpr int kDsWarps = kDsThreads / 32;

struct DsArgs {
  int64_t n_rows, nb, ntiles;
  int64_t full_tiles;
  int serial_blocks;
  VbsDesc d;
  Leg A, B;
  uint32_t* out;
  unsigned long long* count;
};

// Compare the 32 swizzled bytes of a block against literal bytes; GA/EA/GB/EB
// select which of (gt, ge) per leg are computed.  Not computed: gt = 0 (the
// literal byte is 0xFF, nothing is greater), ge = all (the byte is 0x00).
template <bool GA, bool EA, bool GB, bool EB>
__device__ __forceinline__ void cmp_sel(const uint32_t (&w)[8], LevelLit A, LevelLit B,
                                        uint32_t& gtA, uint32_t& geA, uint32_t& gtB,
                                        uint32_t& geB) {
  uint32_t ga = 0, ea = 0, gb = 0, eb = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ev = __byte_perm(w[i], 0, 0x4240);
    const uint32_t od = __byte_perm(w[i], 0, 0x4341);
    if (GA) ga += __byte_perm(ev + A.cgt, od + A.cgt, 0x7351) << i;
    if (EA) ea += __byte_perm(ev + A.cge, od + A.cge, 0x7351) << i;
    if (GB) gb += __byte_perm(ev + B.cgt, od + B.cgt, 0x7351) << i;
    if (EB) eb += __byte_perm(ev + B.cge, od + B.cge, 0x7351) << i;
  }
  gtA = GA ? ga : 0u;
  geA = EA ? ea : kFull;
  gtB = GB ? gb : 0u;
  geB = EB ? eb : kFull;
}

// literal byte class: 0 = other, 1 = 0xFF (no gt), 2 = 0x00 (ge = all)
__device__ __forceinline__ int byte_class(uint32_t b) { return b == 0xFFu ? 1 : (b == 0u ? 2 : 0); }

// (gt, eq) of both legs at level index j0 (0-based) -- eq = ge & ~gt.
template <bool BETWEEN>
__device__ __forceinline__ void cmp_level(const uint32_t (&w)[8], const Leg& A, const Leg& B,
                                          int j0, uint32_t& gA, uint32_t& eA, uint32_t& gB,
                                          uint32_t& eB) {
  const uint32_t ba = A.byte[j0], bb = B.byte[j0];
  const LevelLit la = A.lv[j0], lb = B.lv[j0];
  uint32_t geA, geB;
  if (!BETWEEN || ba == bb) {
    switch (byte_class(ba)) {
      case 1: cmp_sel<false, true, false, false>(w, la, la, gA, geA, gB, geB); break;
      case 2: cmp_sel<true, false, false, false>(w, la, la, gA, geA, gB, geB); break;
      default: cmp_sel<true, true, false, false>(w, la, la, gA, geA, gB, geB); break;
    }
    gB = gA;
    geB = geA;
  } else {
    switch (byte_class(ba) * 3 + byte_class(bb)) {
      case 0: cmp_sel<true, true, true, true>(w, la, lb, gA, geA, gB, geB); break;
      case 1: cmp_sel<true, true, false, true>(w, la, lb, gA, geA, gB, geB); break;
      case 2: cmp_sel<true, true, true, false>(w, la, lb, gA, geA, gB, geB); break;
      case 3: cmp_sel<false, true, true, true>(w, la, lb, gA, geA, gB, geB); break;
      case 5: cmp_sel<false, true, true, false>(w, la, lb, gA, geA, gB, geB); break;
      case 6: cmp_sel<true, false, true, true>(w, la, lb, gA, geA, gB, geB); break;
      case 7: cmp_sel<true, false, false, true>(w, la, lb, gA, geA, gB, geB); break;
      default: cmp_sel<true, true, true, true>(w, la, lb, gA, geA, gB, geB); break;
    }
  }
  eA = geA & ~gA;
  eB = geB & ~gB;
}

template <bool BETWEEN, bool L1, int ST>
__global__ void __launch_bounds__(kDsThreads, 4) vbs_ds_kernel(const __grid_constant__ DsArgs a) {
  constexpr int kRd = ST * 32 + 8;  // deep blocks touched by a super-tile (+ guard)
  __shared__ uint32_t rd_all[kDsWarps][kRd];
  uint32_t* rd = rd_all[threadIdx.x >> 5];
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

  // level-1 sector (L1 only) and M_2 word of block b; zeros past the column
  auto fetch = [&](int64_t b, uint32_t (&w)[8], uint32_t& m2) {
    const bool in = b < a.nb;
    if (L1) {
      if (in) {
        ldg256(d.bs1 + b * 32, w);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = 0;
      }
    }
    m2 = in ? __ldg(d.exist[1] + b) : 0u;
  };
  auto valid_of = [&](int64_t tile, int64_t b) -> uint32_t {
    return tile < a.full_tiles ? kFull : (tile < a.ntiles ? tail_valid(b, a.n_rows) : 0u);
  };

  int64_t st = warp;
  uint32_t wN[8];
  uint32_t m2N = 0;
  if (st < nsuper) fetch(st * ST * 32 + lane, wN, m2N);
  for (; st < nsuper; st += nwarps) {
    const int64_t dfirst = __ldg(d.dir[1] + st * ST * 32);  // first deep row of the super-tile
    uint32_t rs[ST], m2s[ST];
    int offs[ST];
    int soff = 0;  // deep rows of this super-tile so far
    // ---------------- phase 1: shallow rows (lane = row block)
#pragma unroll
    for (int u = 0; u < ST; ++u) {
      const int64_t tile = st * ST + u;
      const int64_t b = tile * 32 + lane;
      uint32_t w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = wN[i];
      const uint32_t m2 = m2N;
      const int64_t ntile = (u + 1 < ST) ? tile + 1 : (st + nwarps) * ST;
      fetch(ntile * 32 + lane, wN, m2N);  // zeros past the column
      uint32_t res = 0;
      if (L1) {
        const uint32_t valid = valid_of(tile, b);
        uint32_t gA, eA, gB, eB;
        cmp_level<BETWEEN>(w, A, B, 0, gA, eA, gB, eB);
        if (BETWEEN) {
          res = valid & (lenA == 1 ? (gA | eA) : gA) & ~gB;
        } else {
          res = finalize_op(A.op, gA, lenA == 1 ? eA : 0u, valid);
        }
        res &= ~m2;
      }
      rs[u] = res;
      m2s[u] = m2;
      const int c2 = __popc(m2);
      const uint32_t incl = warp_incl_scan((uint32_t)c2);
      offs[u] = soff + (int)(incl - (uint32_t)c2);
      soff += (int)__shfl_sync(kFull, incl, 31);
    }
    // ---------------- phase 2: deep rows (lane = deep block)
    const int64_t db0 = dfirst >> 5;
    const int sh0 = (int)(dfirst & 31);
    const int ndt = (sh0 + soff + 31) >> 5;
    for (int t0 = 0; t0 < ndt; t0 += 32) {
      const int t = t0 + lane;
      const bool has = t < ndt;
      const int64_t dbk = db0 + t;
      uint32_t zA = has ? kFull : 0u, zB = (BETWEEN && has) ? kFull : 0u;
      uint32_t gtA = 0, eqA = 0, gtB = 0, eqB = 0;
#pragma unroll
      for (int j = 1; j <= kMaxLevels; ++j) {
        if (j > maxlen) break;
        const bool act = BETWEEN ? ((zA | zB) != 0) : (zA != 0);
        if (!__any_sync(kFull, act)) break;
        uint32_t w[8];
        if (act) {
          ldg256(d.deep[j - 1] + dbk * 32, w);
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = 0;
        }
        // existence of byte j+1 among the deep rows (byte 2 always exists)
        const uint32_t nxt = j >= K ? 0u : (j == 1 ? kFull : (act ? __ldg(d.rexist[j] + dbk) : 0u));
        uint32_t gA, eA, gB, eB;
        cmp_level<BETWEEN>(w, A, B, j - 1, gA, eA, gB, eB);
        vbs_transition(j, lenA, K, gA, eA, nxt, zA, gtA, eqA);
        if (BETWEEN) {
          vbs_transition(j, lenB, K, gB, eB, nxt, zB, gtB, eqB);
          zB &= zA | gtA | eqA;  // hi-leg ties that already fail GE(lo) are settled
        }
      }
      if (has) rd[t] = BETWEEN ? ((gtA | eqA) & ~gtB) : finalize_op(A.op, gtA, eqA, kFull);
    }
    if (lane == 0) rd[ndt] = 0u;  // guard word of the last window
    __syncwarp();
    // ---------------- phase 3: deep results back to row space (lane = row block)
#pragma unroll
    for (int u = 0; u < ST; ++u) {
      const int64_t tile = st * ST + u;
      const int64_t b = tile * 32 + lane;
      const uint32_t m2 = m2s[u];
      const int o = sh0 + offs[u];
      const int wi = o >> 5, sb = o & 31;
      const int c2 = __popc(m2);
      const uint32_t lowm = c2 >= 32 ? kFull : ((1u << c2) - 1u);
      const uint32_t x = c2 ? (__funnelshift_r(rd[wi], rd[wi + 1], sb) & lowm) : 0u;
      uint32_t e = x ? m2 : 0u;
      const bool ntr = x != 0u && x != lowm;
      const uint32_t ntm = __ballot_sync(kFull, ntr);
      if (ntm) {
        if (__popc(ntm) > a.serial_blocks) {
          if (ntr) e = expand_apply(expand_setup(m2), x);
        } else {
          for (uint32_t r = ntm; r; r &= r - 1) {
            const int L = __ffs(r) - 1;
            const uint32_t y =
                warp_pdep(__shfl_sync(kFull, m2, L), __shfl_sync(kFull, x, L), lane);
            if (lane == L) e = y;
          }
        }
      }
      const uint32_t res = rs[u] | e;
      if (b < a.nb) a.out[b] = res;
      cnt += __popc(res);
    }
    __syncwarp();
  }
#pragma unroll
  for (int dd = 16; dd > 0; dd >>= 1) cnt += __shfl_xor_sync(kFull, cnt, dd);
  if (lane == 0 && cnt) atomicAdd(a.count, cnt);
}

template <bool BETWEEN, bool L1, int ST>
static int launch_ds_k(const DsArgs& a, cudaStream_t s) {
  auto kern = vbs_ds_kernel<BETWEEN, L1, ST>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDsThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t nsuper = (a.ntiles + ST - 1) / ST;
  const int64_t want = (nsuper + kDsWarps - 1) / kDsWarps;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  kern<<<grid, kDsThreads, 0, s>>>(a);
  BSB_LAUNCH_CHECK();
  return BSB_OK;
}

template <bool BETWEEN, bool L1>
static int launch_ds(const DsArgs& a, int st, cudaStream_t s) {
  switch (st) {
    case 1: return launch_ds_k<BETWEEN, L1, 1>(a, s);
    case 2: return launch_ds_k<BETWEEN, L1, 2>(a, s);
    case 3: return launch_ds_k<BETWEEN, L1, 3>(a, s);
    default: return launch_ds_k<BETWEEN, L1, 4>(a, s);
  }
}

// Unmasked scan of a SLICED column that carries deep[0].  Returns
// BSB_EINVAL when the column lacks deep[0] (caller falls back).
int vbs_ds_scan(const VbsDesc& d, int64_t n_rows, int64_t deep_rows, const Leg& A,
                const Leg& B, bool between, uint32_t* out, unsigned long long* count,
                cudaStream_t s) {
  DsArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n_rows = n_rows;
  a.nb = (n_rows + 31) / 32;
  a.ntiles = (a.nb + 31) / 32;
  a.full_tiles = n_rows / kTileRows;
  static int serial = -1, st_env = -1;
  if (serial < 0) {
    const char* e = std::getenv("BSB_DS_SERIAL");
    serial = e ? std::atoi(e) : 6;
    const char* t = std::getenv("BSB_DS_TILES");
    st_env = t ? std::atoi(t) : 0;
  }
  a.serial_blocks = serial;
  a.d = d;
  a.A = A;
  a.B = B;
  a.out = out;
  a.count = count;
  // tiles per super-tile: about 28 deep blocks per phase-2 pass
  int st = st_env;
  if (st < 1 || st > 4) {
    const double per_tile = 32.0 * (double)deep_rows / (double)(n_rows > 0 ? n_rows : 1);
    st = per_tile > 0 ? (int)(28.0 / per_tile + 0.5) : 4;
    st = st < 1 ? 1 : (st > 4 ? 4 : st);
  }
  // shallow rows can only match when the level-1 compare can tell them apart
  const bool l1 = between ? !(A.len >= 2 && A.byte[0] == B.byte[0])
                          : !(A.op == BSB_EQ && A.len >= 2);
  BSB_CUDA(cudaMemsetAsync(count, 0, 8, s));
  if (between) return l1 ? launch_ds<true, true>(a, st, s) : launch_ds<true, false>(a, st, s);
  return l1 ? launch_ds<false, true>(a, st, s) : launch_ds<false, false>(a, st, s);
}

}  // namespace bsb
