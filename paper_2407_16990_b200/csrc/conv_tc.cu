// tcgen05 implicit-GEMM 3x3 convolution over packed bins (sm_100a), readings D8/D11 of DESIGN.md.
//
// Layout: activations [bin][row][C/8][Wr][8] bf16 (net.cuh). One bin row of all planes is one
// contiguous run; G consecutive rows are loaded with one cp.async.bulk into an SMEM group slot with
// the same layout, which IS a K-major no-swizzle UMMA operand: pixel m of a core matrix at +16 B, the
// two K-chunks of an MMA at +LBO (= plane stride), so a dx tap is a +-16 B start-address offset.
//
// Mapping ("sliding window"): M = 128 pixels of a row (a tile; a row has T = Wr/128 tiles). The
// three kernel rows are folded into N: one MMA per (dx, K-chunk pair) with N = 3*CP reads input row
// r ONCE and adds its contributions to output rows r+1, r, r-1 together. Output-row accumulators sit
// in TMEM at DEcreasing column addresses (a ring of R slots of CP columns), so those three rows are
// one contiguous 3*CP window (split in two MMAs where it wraps). Every conv uses it, the upsampler
// included, in N chunks of CP <= 85 output columns. SMEM operand traffic per MMA is 4 KB of A +
// 3*CP*32 B of B (measured SS rate: N=96 56 cyc vs 48 ideal, N>=128 at the ideal rate), vs 4 KB of
// A per N=CP MMA for the 9-taps-in-K mapping (N=32: 46 cyc vs 16 ideal).
//
// The single issuing thread must not branch or wait between MMAs (measured: each mbarrier wait
// costs ~100 cycles and every taken branch stalls the issue), so a work unit (bin, band of BR = 32
// output rows, N chunk) is one fully unrolled straight-line MMA sequence over BR + 2 input rows,
// synchronised per group of G rows only: one in_full wait, one acc_empty wait, one in_empty commit,
// one acc_full commit per group. Bands start at an accumulator sequence that is a multiple of R, so
// every TMEM column is a compile-time constant.
//
// Warp roles (320 threads, 1 CTA/SM, persistent over units): warp 0 bulk-copy producer, warp 1 TMEM
// allocator + MMA issuer, warps 2-9 epilogue in two quads taking alternate output-row groups
// (TMEM -> registers -> bias/ReLU/residual/occupancy mask/pixel shuffle -> HBM; row-independent
// loads are issued before the accumulator wait).
#include <stdlib.h>

#include <vector>

#include "fold_common.cuh"
#include "tc_common.cuh"

namespace regen {

namespace tc {

constexpr int NTHREADS = 320;
constexpr int BR = 32;          // output rows per work unit (band)
constexpr int MAX_GSLOTS = 8;   // input group slots in SMEM (power of two)
constexpr int MAX_OG = 8;       // accumulator groups in the TMEM ring (R / G)

struct Params {
  const __nv_bfloat16* in;
  __nv_bfloat16* out;
  const __nv_bfloat16* skip;
  const float* bias;        // [cout] fp32 (original channel order)
  const uint32_t* mbits;    // [bin][bin_h][bin_w/32] occupancy bits
  const int32_t* num_bins;
  const uint8_t* wimg;      // B images, one per N chunk (global)
  uint32_t b_bytes;         // bytes of one chunk's B image
  int Wr, Hr, res, bin_w, bin_h;
  int cout;                 // real output channels of the conv
  int nchunk;               // N chunks
  int nbands;
  int max_bins;
  int out_c8;               // planes of the output activation
  int ngs, gslog;           // input group slots (power of two) and log2
  float res_scale;
  unsigned long long* prof; // optional wait-time counters (REGEN_TC_PROF=1), else null
  int* counter;             // dynamic unit scheduler (zeroed before the launch)
  int reverse;              // hand out units last-to-first (L2 reuse along a conv chain)
  // ROLE_FOLDF only: the fused combine's frame output (fold_common.cuh store_frame)
  const int64_t* fdst;      // [bin][bin_h][bin_w] HR frame index of an owned pixel | rot << 62, else -1
  void* fout;               // HR frames
  const float* tbias;       // tail bias [3]
  int fout_mode, fOW;
  int ff_debug;             // timing experiments only (REGEN_FF_DEBUG): 1 = skip the combine, 2 = skip its stores
  int npr;                  // ROLE_FOLDF: partial-sum rows in the SMEM ring (FF_NPR .. FF_NPR_MAX)
};

// ------------------------------------------------------------------------------- compile-time shape
template <int ROLE, int C, int CP, int R, int G, int T, int PS>
struct Shape {
  // ROLE_FOLDF: a band computes the partial-sum rows y0-1 .. y0+64 (66 rows, one halo row each side)
  // of which the fused combine turns rows y0 .. y0+63 into HR pixels; bands advance by 64 rows
  static constexpr bool FF = ROLE == ROLE_FOLDF;
  static constexpr int BRS = FF ? 66 : BR;                              // output rows computed per band
  static constexpr int BSTR = FF ? 64 : BR;                             // band stride
  static constexpr int ROFF = FF ? -1 : 0;                              // first computed row - band origin
  static constexpr int NT = FF ? NTHREADS + 256 : NTHREADS;             // + 8 combiner warps
  static constexpr bool HEAD = ROLE == ROLE_HEAD || ROLE == ROLE_TINY0;   // Cin = 3, dx packed into K
  static constexpr int KC = HEAD ? 1 : C / 16;                           // K-chunk pairs per dx
  static constexpr int NS = HEAD ? 2 : 3 * KC;                           // MMAs per input row and tile
  static constexpr int N = 3 * CP;
  static constexpr int NG_OUT = BRS / G;                                 // accumulator groups per band
  static constexpr int NG_IN = (BRS + 2 + G - 1) / G;                    // input groups per band
  static constexpr int OGR = R / G;                                      // accumulator groups in the ring
  static constexpr int DONE_LAG = G == 1 ? 2 : 1;                        // input groups until a group completes
  static constexpr bool BIAS_IN_ACC = ROLE != ROLE_UP;                   // slots re-armed with the bias
  static_assert(R % G == 0 && BRS % R == 0 && OGR >= 3 && OGR <= MAX_OG, "ring/group shape");
  static_assert(!FF || (T == 1 && G == 1 && (PS == 2 || PS == 3)), "fused fold: one tile, G = 1");
  static_assert(NG_IN >= NG_OUT + DONE_LAG, "every accumulator group completes inside the band");
  static_assert(T * R * CP <= 512 && N <= 256 && CP % 16 == 0, "TMEM / MMA shape");
  // slot of band-local output row j (accumulator sequence q0 + j, q0 = 0 mod R)
  __host__ __device__ static constexpr int slot(int j) { return (R - (j % R)) % R; }
};

// ------------------------------------------------------------------------------- epilogues
// same-resolution activation (HEAD/RES_A/RES_B/BODY/TINY0): CP output channels, bias in the accumulator
template <int ROLE, int CP>
__device__ __forceinline__ void epi_act(uint32_t taddr, __nv_bfloat16* o, size_t pstride, bool occ, const uint4* sk,
                                        float res_scale) {
  uint32_t r[CP];
#pragma unroll
  for (int c = 0; c < CP; c += 16) tmem_ld16(taddr + (uint32_t)c, r + c);
  tmem_ld_wait();
#pragma unroll
  for (int g = 0; g < CP / 8; ++g) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[8 * g + e]);
    if (ROLE == ROLE_RES_A || ROLE == ROLE_TINY0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
    }
    if (ROLE == ROLE_RES_B || ROLE == ROLE_BODY) {
      const __nv_bfloat162* s2 = reinterpret_cast<const __nv_bfloat162*>(&sk[g]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(s2[e]);
        v[2 * e] = ROLE == ROLE_RES_B ? fmaf(res_scale, v[2 * e], f.x) : v[2 * e] + f.x;
        v[2 * e + 1] = ROLE == ROLE_RES_B ? fmaf(res_scale, v[2 * e + 1], f.y) : v[2 * e + 1] + f.y;
      }
    }
    *reinterpret_cast<uint4*>(o + (size_t)g * pstride) = pack8(v, occ);
  }
}

// upsampler column order: global column n (chunk c = n / CP) -> original output channel (PyTorch
// PixelShuffle order co = ch * PS^2 + sub-position). Chunk c = i * NG + g covers sub-row i and channel
// group g (CG = CP / PS channels); column n % CP = j * CG + e is sub-column j, channel g * CG + e.
template <int C, int CP, int PS>
__host__ __device__ constexpr int up_column(int n) {
  constexpr int CG = CP / PS, NG = C / CG;
  const int c = n / CP, w = n - c * CP;
  const int i = c / NG, g = c - i * NG, j = w / CG, e = w - j * CG;
  return (g * CG + e) * PS * PS + i * PS + j;
}

// ------------------------------------------------------------------------------- kernel
constexpr int FF_NPR = 4;   // ROLE_FOLDF: partial-sum rows held in SMEM for the fused combine (at least 4 x 20.8 KB,
                            // leaving room for an 8-row input ring: the row loads are latency-bound)
constexpr int FF_NPR_MAX = 6;
constexpr int FF_W = 130;   // ring row width: 128 pixels + a zero column each side (the combine's x
                            // padding, so its 16-B loads need no bounds checks)

template <int ROLE, int C, int CP, int R, int G, int T, int PS>
__global__ void __launch_bounds__(ROLE == ROLE_FOLDF ? NTHREADS + 256 : NTHREADS, 1)
    conv_tc_kernel(const __grid_constant__ Params p) {
  using S = Shape<ROLE, C, CP, R, G, T, PS>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t in_full[MAX_GSLOTS], in_empty[MAX_GSLOTS];
  __shared__ __align__(8) uint64_t acc_full[MAX_OG], acc_empty[MAX_OG];
  __shared__ __align__(8) uint64_t b_full[2], b_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(16) float bias_sm[768];   // bias per accumulator column (all chunks)
  __shared__ __align__(8) uint64_t prow_full[FF_NPR_MAX], prow_empty[FF_NPR_MAX];   // ROLE_FOLDF partial-sum rows

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cin8 = S::HEAD ? 1 : C / 8;
  const uint32_t row_bytes = (uint32_t)cin8 * p.Wr * 16;
  const uint32_t grp_bytes = row_bytes * G;
  const uint32_t ngs = (uint32_t)p.ngs, gsm = ngs - 1, gslog = (uint32_t)p.gslog;
  // SMEM: [1 KB guard][ngs x G rows][B image(s)][ROLE_FOLDF: FF_NPR partial-sum rows]
  uint8_t* ring = smem_raw + 1024;
  uint8_t* bimg = ring + ngs * grp_bytes;
  uint8_t* pring = bimg + (p.nchunk > 1 ? 2u : 1u) * p.b_bytes;   // [FF_NPR][CP/8][Wr][16 B]
  constexpr uint32_t PROW_BYTES = (uint32_t)CP / 8 * FF_W * 16;    // T == 1: Wr == 128 (+2 zero columns)
  // units are (bin, band, chunk), chunk fastest (the chunks of a band re-read its input rows from L2),
  // over the bins actually used; B images are double-buffered per unit when there are several chunks.
  // Units are handed out by
  // an atomic counter (the producer) through a small SMEM ring, so CTAs that start late (an SM busy
  // with another stream's kernel) simply take fewer units
  const int nbins = min(*p.num_bins, p.max_bins);
  const int per_chunk = nbins * p.nbands;
  const int total_units = per_chunk * p.nchunk;
  __shared__ int unit_ring[4];
  __shared__ __align__(8) uint64_t unit_full[4], unit_empty[4];

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < (int)ngs; ++i) { mbar_init(&in_full[i], 1); mbar_init(&in_empty[i], 1); }
    for (int i = 0; i < S::OGR; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
    for (int i = 0; i < 2; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 4; ++i) { mbar_init(&unit_full[i], 1); mbar_init(&unit_empty[i], S::FF ? 17 : 9); }
    // a partial-sum row is written by one epilogue quad (128 lane arrivals, each lane releasing its own
    // stores) and read by the three combines of rows r-1, r, r+1 (3 x 128 lane arrivals; band-edge
    // rows get the missing ones from the edge combines)
    if (S::FF)
      for (int i = 0; i < p.npr; ++i) { mbar_init(&prow_full[i], 128); mbar_init(&prow_empty[i], 3 * 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // bias in accumulator-column order: chunk c column n = global column c*CP + n. Upsampler chunks are
  // (sub-row i, channel group g) with columns n = j*CG + e (sub-column j, channel g*CG + e): see
  // up_column() — each chunk then writes whole HR pixels of CG channels for all sub-columns j.
  for (int n = threadIdx.x; n < 768; n += S::NT) {
    float b = 0.f;
    if constexpr (ROLE == ROLE_UP) {
      const int co = up_column<C, CP, PS>(n);
      if (co < p.cout) b = __ldg(p.bias + co);
    } else if (n < p.cout) {
      b = __ldg(p.bias + n);
    }
    bias_sm[n] = b;
  }
  if (S::FF) {   // the ring rows' zero columns (x = -1 and x = 128), never overwritten
    for (int i = threadIdx.x; i < p.npr * (CP / 8) * 2; i += S::NT) {
      const int row = i / ((CP / 8) * 2), r2 = i - row * (CP / 8) * 2, pl = r2 >> 1, side = r2 & 1;
      *reinterpret_cast<uint4*>(pring + row * PROW_BYTES + (uint32_t)(pl * FF_W + side * (FF_W - 1)) * 16) =
          make_uint4(0, 0, 0, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  // arm every accumulator slot: bias (single-chunk convs) or zero (upsampler chunks)
  if (warp >= 2 && warp < 6) {
    const int q4 = warp & 3;
    float z[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) z[e] = 0.f;
    for (int t = 0; t < T; ++t)
      for (int s = 0; s < R; ++s)
#pragma unroll
        for (int c0 = 0; c0 < CP; c0 += 16)
          tmem_st16(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)((t * R + s) * CP + c0),
                    S::BIAS_IN_ACC ? bias_sm + c0 : z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long pw0 = 0, pw1 = 0, pw2 = 0, pw3 = 0, pwS = 0, pwR = 0;   // pwR: ROLE_FOLDF ring waits
  const long long pstart = clock64();

  if (warp == 0) {
    // =============================== producer ===============================
    if (lane == 0) {
      uint32_t ig = 0;          // input groups loaded (ring sequence)
      uint32_t bload = 0;
      for (uint32_t us = 0;; ++us) {
        int u = atomicAdd(p.counter, 1);
        if (u >= total_units) u = -1;
        else if (p.reverse) u = total_units - 1 - u;
        mbar_wait(&unit_empty[us & 3], ((us >> 2) & 1) ^ 1);
        unit_ring[us & 3] = u;
        mbar_arrive(&unit_full[us & 3]);
        if (u < 0) break;
        const int v = u / p.nchunk, chunk = u - v * p.nchunk;
        const int bin = v / p.nbands, y0 = (v - bin * p.nbands) * S::BSTR + S::ROFF;
        if (p.nchunk > 1 || bload == 0) {
          const uint32_t bs = bload & 1;
          mbar_wait(&b_empty[bs], ((bload >> 1) & 1) ^ 1);
          mbar_expect_tx(&b_full[bs], p.b_bytes);
          bulk_g2s(bimg + bs * p.b_bytes, p.wimg + (size_t)chunk * p.b_bytes, p.b_bytes, &b_full[bs]);
          ++bload;
        }
        const int y1 = min(p.Hr, y0 + S::BRS);
        const int rlo = max(y0 - 1, 0), rhi = min(y1, p.Hr - 1);   // input rows this unit reads
        for (int k = 0; k < S::NG_IN; ++k) {
          const uint32_t slot = ig & gsm;
          {
            const long long t0 = clock64();
            mbar_wait(&in_empty[slot], ((ig >> gslog) & 1) ^ 1);
            if (p.prof) pw0 += clock64() - t0;
          }
          const int g0 = y0 - 1 + G * k;                 // input row of group row 0
          const int a = max(g0, rlo), b = min(g0 + G - 1, rhi);
          if (a <= b) {
            mbar_expect_tx(&in_full[slot], (uint32_t)(b - a + 1) * row_bytes);
            bulk_g2s(ring + slot * grp_bytes + (uint32_t)(a - g0) * row_bytes,
                     p.in + ((size_t)bin * p.Hr + a) * (row_bytes / 2), (uint32_t)(b - a + 1) * row_bytes,
                     &in_full[slot]);
          } else {
            mbar_arrive(&in_full[slot]);
          }
          ++ig;
        }
      }
    }
  } else if (warp == 1) {
    // =============================== MMA issuer ===============================
    if (elect_one()) {
      uint32_t ig = 0, og = 0, bwait = 0;
      uint32_t b16 = smem_u32(bimg) >> 4, bs = 0;
      const uint32_t ring16 = smem_u32(ring) >> 4;
      const uint32_t row16 = row_bytes >> 4, grp16 = grp_bytes >> 4;
      const uint32_t plane16 = (uint32_t)p.Wr;              // A plane stride (16-B units)
      constexpr uint32_t BLBO = (uint32_t)S::N;              // B chunk-plane stride (16-B units)
      for (uint32_t us = 0;; ++us) {
        mbar_wait(&unit_full[us & 3], (us >> 2) & 1);
        const int u = *(volatile int*)&unit_ring[us & 3];
        mbar_arrive(&unit_empty[us & 3]);
        if (u < 0) break;
        const int v = u / p.nchunk, chunk = u - v * p.nchunk;
        const int bin = v / p.nbands, y0 = (v - bin * p.nbands) * S::BSTR + S::ROFF;
        if (p.nchunk > 1 || bwait == 0) {
          bs = bwait & 1;
          mbar_wait(&b_full[bs], (bwait >> 1) & 1);
          ++bwait;
          b16 = (smem_u32(bimg) + bs * p.b_bytes) >> 4;
        }
        const int rlo = max(y0 - 1, 0), rhi = min(min(y0 + S::BRS, p.Hr), p.Hr - 1);
#pragma unroll
        for (int k = 0; k < S::NG_IN; ++k) {
          const uint32_t slot = (ig + k) & gsm;
          if (k < S::NG_OUT) {
            const uint32_t og_k = og + k;
            const long long t0 = clock64();
            mbar_wait(&acc_empty[og_k % S::OGR], ((og_k / S::OGR) & 1) ^ 1);
            if (p.prof) pw1 += clock64() - t0;
          }
          {
            const uint32_t igk = ig + k;
            const long long t0 = clock64();
            mbar_wait(&in_full[slot], (igk >> gslog) & 1);
            if (p.prof) pw2 += clock64() - t0;
          }
          tc_fence_after();
          const uint32_t grp_a = ring16 + slot * grp16;
#pragma unroll
          for (int ii = 0; ii < G; ++ii) {
            constexpr int dummy = 0;
            (void)dummy;
            const int i = G * k + ii;                 // band-local input row: r = y0 - 1 + i
            if (i > S::BRS + 1) continue;              // compile-time
            const int r = y0 - 1 + i;
            const uint32_t en = (r >= rlo && r <= rhi) ? 1u : 0u;
            // window: output rows j = i (group 0, dy=-1), i-1 (group 1), i-2 (group 2) inside [0, BR)
            const int gA = i < S::BRS ? 0 : (i - 1 < S::BRS ? 1 : 2);
            const int gB = i >= 2 ? 3 : (i >= 1 ? 2 : 1);
            const int ng = gB - gA;
            const int s0 = S::slot(i - gA);          // slot of the first group's output row
            const int len1 = ng < R - s0 ? ng : R - s0;
            const uint32_t a_row = grp_a + (uint32_t)ii * row16;
#pragma unroll
            for (int t = 0; t < T; ++t) {
              const uint32_t tcol = tmem + (uint32_t)(t * R * CP);
#pragma unroll
              for (int st = 0; st < S::NS; ++st) {
                int dx, plane;
                uint32_t lbo;
                // HEAD: Cin = 3 padded to 8, dx packed into K: step 0 reads pixels x-1, x (kernel columns 0, 1),
                // step 1 pixels x, x+1 (column 2 in the second half, zero weights in the first). Every A row m
                // then reads pixels m-1 .. m+1 only: an occupied pixel (x <= W-2, D8) never reads past its bin
                // row (stale SMEM there could hold NaN patterns, and 0 * NaN = NaN in the MMA)
                if (S::HEAD) { dx = st == 0 ? -1 : 0; plane = 0; lbo = 1; }
                else { dx = st / S::KC - 1; plane = 2 * (st % S::KC); lbo = plane16; }
                const uint32_t a_lo = (a_row + (uint32_t)t * 128u + (uint32_t)plane * plane16 + (uint32_t)dx) +
                                      (lbo << 16);
                const uint32_t b_lo = (b16 + (uint32_t)(st * S::N * 2) + (uint32_t)(gA * CP)) + (BLBO << 16);
                mma_bf16(tcol + (uint32_t)(s0 * CP), a_lo, b_lo, make_idesc(len1 * CP), en);
                if (len1 < ng)
                  mma_bf16(tcol, a_lo, b_lo + (uint32_t)(len1 * CP), make_idesc((ng - len1) * CP), en);
              }
            }
          }
          mma_commit(&in_empty[slot]);                   // input group k consumed
          // accumulator group c is complete once input row G*c + G + 1 has been added (dy = +1 of its
          // last row): after input group c + 1 (G >= 2) or c + 2 (G == 1)
          if (k >= S::DONE_LAG && k - S::DONE_LAG < S::NG_OUT) mma_commit(&acc_full[(og + k - S::DONE_LAG) % S::OGR]);
        }
        if (p.nchunk > 1) mma_commit(&b_empty[bs]);   // this unit's B image can be overwritten
        ig += S::NG_IN;
        og += S::NG_OUT;
      }
    }
    __syncwarp();
  } else if (warp < NTHREADS / 32) {
    // =============================== epilogue ===============================
    const int quad = (warp - 2) >> 2;        // alternate accumulator groups between the two quads
    const int q4 = warp & 3;                 // TMEM lane quarter of this warp
    const int m = 32 * q4 + lane;            // pixel within the tile
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    constexpr bool HAS_SKIP = ROLE == ROLE_RES_B || ROLE == ROLE_BODY;
    constexpr int SK = HAS_SKIP ? CP / 8 : 1;
    const int words = p.bin_w / 32;
    const size_t bin_px = (size_t)p.Hr * p.Wr;
    const size_t pstride = (size_t)p.Wr * 8;                 // elements between planes of one row
    uint32_t og = 0;
    uint32_t pbase = 0;   // ROLE_FOLDF: sequence number of this unit's first partial-sum row
    for (uint32_t us = 0;; ++us) {
      mbar_wait(&unit_full[us & 3], (us >> 2) & 1);
      const int u = *(volatile int*)&unit_ring[us & 3];
      __syncwarp();
      if (lane == 0) mbar_arrive(&unit_empty[us & 3]);
      if (u < 0) break;
      const int v = u / p.nchunk, chunk = u - v * p.nchunk;
      const int bin = v / p.nbands, y0 = (v - bin * p.nbands) * S::BSTR + S::ROFF;
      const int nrows = min(S::BRS, p.Hr - y0);
      // one tile per row (T == 1): the occupancy words of all the band's rows for this warp's 32 pixels
      // (one word: 32 pixels at res 1, 64 at res 2) are fetched once per unit, <= 3 per lane, and handed
      // to each row by a shuffle, so no per-row global-load latency sits on the epilogue's path
      uint32_t occ_pre[3] = {0u, 0u, 0u};
      if constexpr (T == 1) {
        const int wq = ((32 * q4) / p.res) / 32;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int r = 32 * q + lane;
          const int y = min(max(y0 + r, 0), p.Hr - 1);
          if (r < S::BRS) occ_pre[q] = __ldg(p.mbits + ((size_t)bin * p.bin_h + y / p.res) * words + wq);
        }
      }
      for (int k = 0; k < S::NG_OUT; ++k) {
        const uint32_t og_k = og + k;
        if ((int)(og_k & 1) != quad) continue;
        // row-independent loads for all rows of the group, issued before the accumulator wait
        const int ybase = y0 + G * k;
        uint32_t occw[G][T];
        uint4 sk[G][SK];
#pragma unroll
        for (int jj = 0; jj < G; ++jj) {
          const int y = min(max(ybase + jj, 0), p.Hr - 1);
          const uint32_t* mrow = p.mbits + ((size_t)bin * p.bin_h + y / p.res) * words;
          if constexpr (T == 1) {
            const int r = G * k + jj;   // band-local row; shuffle the prefetched word (warp-uniform r)
            const uint32_t w01 = r < 32 ? occ_pre[0] : occ_pre[1];
            occw[jj][0] = __shfl_sync(0xffffffffu, r < 64 ? w01 : occ_pre[2], r & 31);
            (void)mrow;
          } else {
#pragma unroll
            for (int t = 0; t < T; ++t) occw[jj][t] = __ldg(mrow + ((t * 128 + m) / p.res) / 32);
          }
          if (HAS_SKIP) {
            const size_t act_row = (size_t)bin * bin_px * p.out_c8 * 8 + (size_t)y * p.out_c8 * pstride;
#pragma unroll
            for (int g = 0; g < SK; ++g)
              sk[jj][g] = *reinterpret_cast<const uint4*>(p.skip + act_row + (size_t)g * pstride + (size_t)m * 8);
          }
        }
        {
          const long long t0 = clock64();
          mbar_wait(&acc_full[og_k % S::OGR], (og_k / S::OGR) & 1);
          if (p.prof) pw3 += clock64() - t0;
        }
        tc_fence_after();
#pragma unroll
        for (int jj = 0; jj < G; ++jj) {
          const int j = G * k + jj;
          const int y = y0 + j;
          if constexpr (S::FF) {
            // partial-sum row j -> SMEM ring (bf16, masked: exactly the values ROLE_FOLD writes to
            // HBM); rows outside the bin are zero rows (the combine's zero padding)
            const uint32_t q = pbase + (uint32_t)j;
            const uint32_t sl = q % (uint32_t)p.npr;
            {
              const long long t0 = clock64();
              mbar_wait(&prow_empty[sl], ((q / (uint32_t)p.npr) & 1) ^ 1);
              if (p.prof) pwR += clock64() - t0;
            }
            uint8_t* rowp = pring + sl * PROW_BYTES + (uint32_t)(m + 1) * 16;
            if (y >= 0 && y < p.Hr) {
              const bool occ = (occw[jj][0] >> (m & 31)) & 1u;
              const uint32_t taddr = tmem + lane_off + (uint32_t)(S::slot(j) * CP);
              // two batches of TMEM columns (<= 48 live registers: no spills beside the r[] of 80)
              constexpr int H1 = CP / 16 / 2 * 16 + (CP / 16 % 2) * 16;   // 48 of 80, 32 of 48
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c0 = h ? H1 : 0, c1 = h ? CP : H1;
                uint32_t r[H1];
#pragma unroll
                for (int c = 0; c < H1; c += 16) {
                  if (c0 + c >= c1) continue;
                  if (PS == 3 && c0 + c == 64) {   // 75 partial channels of 80: columns 64..74 only
                    tmem_ld8(taddr + 64u, r + c);
                    tmem_ld2(taddr + 72u, r + c + 8);
                    tmem_ld1(taddr + 74u, r + c + 10);
#pragma unroll
                    for (int e = 11; e < 16; ++e) r[c + e] = 0u;   // padding channels, never read
                  } else {
                    tmem_ld16(taddr + (uint32_t)(c0 + c), r + c);
                  }
                }
                tmem_ld_wait();
#pragma unroll
                for (int g = 0; g < H1 / 8; ++g) {
                  if (c0 + 8 * g >= c1) break;
                  float vv[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) vv[e] = __uint_as_float(r[8 * g + e]);
                  *reinterpret_cast<uint4*>(rowp + (c0 / 8 + g) * FF_W * 16) = pack8(vv, occ);
                }
              }
            } else {
#pragma unroll
              for (int g = 0; g < CP / 8; ++g) *reinterpret_cast<uint4*>(rowp + g * FF_W * 16) = make_uint4(0, 0, 0, 0);
            }
            mbar_arrive(&prow_full[sl]);   // every writer lane releases its own row stores
          } else if (j < nrows) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
              const int x = t * 128 + m;
              const int xl = x / p.res;
              const bool occ = (occw[jj][t] >> (xl & 31)) & 1u;
              const uint32_t taddr = tmem + lane_off + (uint32_t)((t * R + S::slot(j)) * CP);
              if constexpr (ROLE == ROLE_TAIL) {
                uint32_t r[16];
                tmem_ld16(taddr, r);
                tmem_ld_wait();
                uint2 val;
                val.x = pack_bf16x2(occ ? __uint_as_float(r[0]) : 0.f, occ ? __uint_as_float(r[1]) : 0.f);
                val.y = pack_bf16x2(occ ? __uint_as_float(r[2]) : 0.f, 0.f);
                *reinterpret_cast<uint2*>(p.out + ((size_t)bin * bin_px + (size_t)y * p.Wr + x) * 4) = val;
              } else if constexpr (ROLE == ROLE_UP) {
                // chunk = (sub-row i, channel group g): + bias, PixelShuffle(PS) into [bin][Y][C/8][X][8];
                // per plane the PS sub-columns of a pixel are adjacent 16-B chunks (full sectors)
                constexpr int CG = CP / PS, NG = C / CG;
                const int i2 = chunk / NG, g2 = chunk - i2 * NG;
                const int Wo = p.Wr * PS;
                __nv_bfloat16* orow = p.out + (size_t)bin * bin_px * PS * PS * C +
                                      (size_t)(y * PS + i2) * (C / 8) * Wo * 8 + (size_t)(x * PS) * 8;
                uint32_t r[CP];
#pragma unroll
                for (int c = 0; c < CP; c += 16) tmem_ld16(taddr + (uint32_t)c, r + c);
                tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < CG / 8; ++q) {
                  __nv_bfloat16* o = orow + (size_t)(g2 * (CG / 8) + q) * Wo * 8;
#pragma unroll
                  for (int j2 = 0; j2 < PS; ++j2) {
                    const int cl = j2 * CG + 8 * q;      // column within the chunk
                    float vv[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) vv[e] = __uint_as_float(r[cl + e]) + bias_sm[chunk * CP + cl + e];
                    *reinterpret_cast<uint4*>(o + j2 * 8) = pack8(vv, occ);
                  }
                }
              } else {
                const size_t act = (size_t)bin * bin_px * p.out_c8 * 8 + (size_t)y * p.out_c8 * pstride + (size_t)x * 8;
                uint4 skt[SK];
#pragma unroll
                for (int g = 0; g < SK; ++g)
                  skt[g] = (HAS_SKIP && t > 0) ? *reinterpret_cast<const uint4*>(p.skip + act + (size_t)g * pstride)
                                               : sk[jj][g];
                epi_act<ROLE, CP>(taddr, p.out + act, pstride, occ, skt, p.res_scale);
              }
            }
          }
          // re-arm the group's slots (all tiles) for their next use
          const long long tst = clock64();
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const uint32_t taddr = tmem + lane_off + (uint32_t)((t * R + S::slot(j)) * CP);
            float z[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) z[e] = 0.f;
#pragma unroll
            for (int c = 0; c < CP; c += 16) {
              if (S::FF && PS == 3 && c == 64) {   // the 5 padding columns accumulate zeros: never re-armed
                tmem_st8(taddr + 64u, bias_sm + 64);
                tmem_st2(taddr + 72u, bias_sm + 72);
                tmem_st1(taddr + 74u, bias_sm + 74);
              } else {
                tmem_st16(taddr + (uint32_t)c, S::BIAS_IN_ACC ? bias_sm + c : z);
              }
            }
          }
          if (p.prof) pwS += clock64() - tst;
        }
        {
          const long long t0 = clock64();
          tmem_st_wait();
          if (p.prof) pwS += clock64() - t0;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[og_k % S::OGR]);
      }
      og += S::NG_OUT;
      pbase += S::BRS;
    }
  } else {
    // =============================== fused combine (ROLE_FOLDF) ===============================
    // Two groups of 4 warps take alternate band rows c (group 0 odd, group 1 even); a thread per bin
    // pixel column x of the (single) tile. For band row c (bin row yb + c - 1) a group waits for the
    // partial-sum rows c-1, c, c+1, sums the <= 4 partials of each HR sub-pixel exactly as the
    // standalone combine does (fold_common.cuh), writes the owned pixel's HR block into the frame and
    // then signals that it has read the three rows (a row's slot is free after all three readers).
    if constexpr (S::FF) {
      const int cw = warp - NTHREADS / 32;          // 0..7
      const int grp = cw >> 2;
      const int x = (cw & 3) * 32 + lane;
      const float b0 = __ldg(p.tbias), b1 = __ldg(p.tbias + 1), b2 = __ldg(p.tbias + 2);
      uint32_t pbase = 0;
      for (uint32_t us = 0;; ++us) {
        mbar_wait(&unit_full[us & 3], (us >> 2) & 1);
        const int u = *(volatile int*)&unit_ring[us & 3];
        __syncwarp();
        if (lane == 0) mbar_arrive(&unit_empty[us & 3]);
        if (u < 0) break;
        const int bin = u / p.nbands, yb = (u - bin * p.nbands) * S::BSTR;   // nchunk == 1
        const int64_t* drow = p.fdst + (size_t)bin * p.bin_h * p.bin_w + x;
        // first row of this group: c0 = 1 (group 0) or 2 (group 1); the frame destination of the next
        // row is loaded one row ahead (L2 latency off the chain)
        const int c0 = grp ? 2 : 1;
        int64_t dnext = yb + c0 - 1 < p.Hr ? __ldg(drow + (size_t)(yb + c0 - 1) * p.bin_w) : -1;
#pragma unroll 1
        for (int c = c0; c <= S::BSTR; c += 2) {
          const int y = yb + c - 1;
          const int64_t dst = dnext;
          dnext = (c + 2 <= S::BSTR && y + 2 < p.Hr) ? __ldg(drow + (size_t)(y + 2) * p.bin_w) : -1;
          const uint8_t* rb[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const uint32_t q = pbase + (uint32_t)(c - 1 + d);
            const long long t0 = clock64();
            mbar_wait(&prow_full[q % (uint32_t)p.npr], (q / (uint32_t)p.npr) & 1);
            if (p.prof) pwR += clock64() - t0;
            rb[d] = pring + (q % (uint32_t)p.npr) * PROW_BYTES + (uint32_t)(x + 1) * 16;
          }
          if (y < p.Hr && dst >= 0 && p.ff_debug != 1) {
            float acc[PS][PS][3];
            fold::accumulate_batched<PS, 6>(
                [&](int l) {
                  const int ny = fold::load_ny(PS, l), nx = fold::load_nx(PS, l), pl = fold::load_pl(PS, l);
                  return *reinterpret_cast<const uint4*>(rb[ny + 1] + (pl * FF_W + nx) * 16);
                },
                acc);
            if (p.ff_debug != 2)   // 2: compute but skip the frame stores (timing experiments only)
              fold::store_frame<PS>(acc, b0, b1, b2, dst, 1, x, y, p.fOW, p.fout, p.fout_mode);
            else {   // keep every accumulator live
              float cs = 0.f;
#pragma unroll
              for (int i = 0; i < PS; ++i)
#pragma unroll
                for (int j = 0; j < PS; ++j) cs += acc[i][j][0] + acc[i][j][1] + acc[i][j][2];
              if (cs == 1234.5f) *(volatile float*)p.fout = cs;
            }
          }
          {   // every combiner lane releases its own reads of the three rows
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              // row c-1+d read once by this combine; the band-edge rows 0, 1, 64, 65 also take the
              // arrivals of the combines that do not exist (c = 0, c = 65)
              uint32_t n = 1;
              if (c == 1 && d == 0) n = 3;
              if (c == 1 && d == 1) n = 2;
              if (c == S::BSTR && d == 1) n = 2;
              if (c == S::BSTR && d == 2) n = 3;
              mbar_arrive_cnt(&prow_empty[(pbase + (uint32_t)(c - 1 + d)) % (uint32_t)p.npr], n);
            }
          }
        }
        pbase += S::BRS;
      }
    }
  }
  if (p.prof && lane == 0) {
    const long long tot = clock64() - pstart;
    if (warp == 0) { atomicAdd(p.prof + 0, (unsigned long long)pw0); atomicAdd(p.prof + 4, (unsigned long long)tot); }
    if (warp == 1) { atomicAdd(p.prof + 1, (unsigned long long)pw1); atomicAdd(p.prof + 2, (unsigned long long)pw2);
                     atomicAdd(p.prof + 5, (unsigned long long)tot); }
    if (warp >= 2 && warp < NTHREADS / 32) {
      atomicAdd(p.prof + 3, (unsigned long long)pw3); atomicAdd(p.prof + 6, (unsigned long long)tot);
      atomicAdd(p.prof + 7, (unsigned long long)pwS); atomicAdd(p.prof + 8, (unsigned long long)pwR);
    }
    if (warp >= NTHREADS / 32) { atomicAdd(p.prof + 9, (unsigned long long)pwR); atomicAdd(p.prof + 10, (unsigned long long)tot); }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------- host plans
struct Plan {
  bool ok = false;
  int cp = 0, nchunk = 1, R = 0, G = 0, T = 0, ns = 0;
  uint32_t b_bytes = 0;
};

static uint16_t bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// W index in the caller's layout [cout][cin][3][3]
static inline float wv(const float* W, int cin, int co, int ci, int ky, int kx) {
  return W[(((size_t)co * cin + ci) * 3 + ky) * 3 + kx];
}

// ring shape for CP columns per slot, T tiles and a row of row_bytes: the largest power-of-two R
// with T*R*CP <= 512, then the largest group G in {4, 2, 1} with >= 3 accumulator groups in the ring
// (R/G >= 3, so the epilogue drains one group while the MMAs fill the next two) and >= 2 input group
// slots of G rows in SMEM next to the B image.
static bool ring_shape(int CP, int T, uint32_t row_bytes, uint32_t b_bytes, int& R, int& G) {
  R = 16;
  while (R > 4 && T * R * CP > 512) R >>= 1;
  if (T * R * CP > 512) return false;
  for (int g : {4, 2, 1}) {
    if (R / g >= 3 && R / g <= MAX_OG && 1024 + 2ull * g * row_bytes + b_bytes <= 220 * 1024) {
      G = g;
      return true;
    }
  }
  return false;
}

// B image of one N chunk: per step st (dx-major, then K-chunk pair), a block [2 K-chunks][3*CP rows][8]
// bf16 (K-major, no swizzle, SBO 128, LBO 3*CP*16); row g*CP + n = kernel row ky = g, chunk column n.
static bool plan_conv(const ConvDesc& d, int C, int res, int bin_w, Plan& pl, std::vector<uint16_t>& img,
                      const float* W) {
  const bool head = d.cin == 3;
  if (d.role == ROLE_TINY1) return false;          // 3 channels per sub-position: SIMT kernel
  if (!head && d.cin != C) return false;
  if (C % 16 != 0) return false;
  const int Wr = bin_w * res;
  if (Wr % 128 != 0 || bin_w % 32 != 0) return false;
  pl.T = Wr / 128;
  if (pl.T > 4) return false;
  int CP = 0;
  const uint32_t row_bytes = (uint32_t)(head ? 1 : d.cin / 8) * Wr * 16;
  const int kc = head ? 1 : d.cin / 16, nsteps = head ? 2 : 3 * kc;
  if (d.role == ROLE_UP) {
    // chunk = (sub-row, group of CG channels x PS sub-columns): CP = PS * CG
    for (int cg : {32, 16}) {
      const int cand = d.ps * cg;
      if (C % cg == 0 && 3 * cand <= 256 && cand % 16 == 0 &&
          ring_shape(cand, pl.T, row_bytes, (uint32_t)(nsteps * 3 * cand * 32), pl.R, pl.G)) {
        CP = cand;
        break;
      }
    }
    if (CP == 0) return false;
  } else {
    CP = (d.cout + 15) / 16 * 16;
    if (3 * CP > 256) return false;
    if (!ring_shape(CP, pl.T, row_bytes, (uint32_t)(nsteps * 3 * CP * 32), pl.R, pl.G)) return false;
  }
  pl.cp = CP;
  pl.nchunk = d.role == ROLE_UP ? d.cout / CP : 1;
  const int N = 3 * CP;
  const int KC = head ? 1 : d.cin / 16;
  pl.ns = head ? 2 : 3 * KC;
  const size_t chunk_elems = (size_t)pl.ns * N * 16;
  img.assign(chunk_elems * pl.nchunk, 0);
  const int s2 = d.ps * d.ps;
  for (int j = 0; j < pl.nchunk; ++j)
    for (int st = 0; st < pl.ns; ++st) {
      const size_t base = j * chunk_elems + (size_t)st * N * 16;
      for (int g = 0; g < 3; ++g)
        for (int n = 0; n < CP; ++n) {
          int co;
          if (d.role == ROLE_UP) {
            const int col = j * CP + n, cg = CP / d.ps, ng = C / cg;
            const int cc = col / CP, w = col - cc * CP, i = cc / ng, gg = cc - i * ng, jj = w / cg, e = w - jj * cg;
            co = (gg * cg + e) * s2 + i * d.ps + jj;
          } else {
            co = n;
          }
          if (co >= d.cout) continue;
          for (int k = 0; k < 16; ++k) {
            float v = 0.f;
            if (head) {
              const int dx = st == 0 ? (k < 8 ? -1 : 0) : (k < 8 ? 99 : 1);   // 99: zero weight
              const int ci = k % 8;
              if (dx != 99 && ci < 3) v = wv(W, 3, co, ci, g, dx + 1);
            } else {
              const int dx = st / KC - 1, ci = 16 * (st % KC) + k;
              v = wv(W, d.cin, co, ci, g, dx + 1);
            }
            img[base + (size_t)(k / 8) * N * 8 + (size_t)(g * CP + n) * 8 + (k % 8)] = bf16_bits(v);
          }
        }
    }
  pl.b_bytes = (uint32_t)(chunk_elems * 2);
  pl.ok = true;
  return true;
}

struct NetPlans {
  std::vector<Plan> plans;   // per conv; !ok => SIMT
};

typedef void (*KernFn)(Params);

template <int ROLE, int C, int CP, int R, int G, int T, int PS>
static KernFn kfn() {
  return conv_tc_kernel<ROLE, C, CP, R, G, T, PS>;
}

// instance table: every (role, C, CP, R, G, T, PS) the planner can produce for C in {16, 32, 48, 64}
static KernFn lookup(int role, int C, int CP, int R, int G, int T, int PS) {
#define K(ROLE_, C_, CP_, R_, G_, T_, PS_)                                                                 \
  if (role == ROLE_ && C == C_ && CP == CP_ && R == R_ && G == G_ && T == T_ && PS == PS_)                \
    return kfn<ROLE_, C_, CP_, R_, G_, T_, PS_>();
  K(ROLE_BODY, 16, 16, 16, 4, 1, 1)
  K(ROLE_HEAD, 16, 16, 16, 4, 1, 1)
  K(ROLE_RES_A, 16, 16, 16, 4, 1, 1)
  K(ROLE_RES_B, 16, 16, 16, 4, 1, 1)
  K(ROLE_TAIL, 16, 16, 16, 4, 2, 1)
  K(ROLE_TAIL, 16, 16, 8, 2, 3, 1)
  K(ROLE_TAIL, 16, 16, 8, 2, 4, 1)
  K(ROLE_TINY0, 16, 16, 16, 4, 1, 1)
  K(ROLE_UP, 16, 32, 16, 4, 1, 2)
  K(ROLE_UP, 16, 32, 8, 2, 2, 2)
  K(ROLE_UP, 16, 48, 8, 2, 1, 3)
  K(ROLE_BODY, 32, 32, 16, 4, 1, 1)
  K(ROLE_HEAD, 32, 32, 16, 4, 1, 1)
  K(ROLE_RES_A, 32, 32, 16, 4, 1, 1)
  K(ROLE_RES_B, 32, 32, 16, 4, 1, 1)
  K(ROLE_TAIL, 32, 16, 16, 4, 2, 1)
  K(ROLE_TAIL, 32, 16, 8, 2, 3, 1)
  K(ROLE_TAIL, 32, 16, 8, 2, 4, 1)
  K(ROLE_TINY0, 32, 32, 16, 4, 1, 1)
  K(ROLE_UP, 32, 48, 8, 2, 1, 3)
  K(ROLE_UP, 32, 64, 8, 2, 1, 2)
  K(ROLE_UP, 32, 64, 4, 1, 2, 2)
  K(ROLE_BODY, 48, 48, 8, 2, 1, 1)
  K(ROLE_HEAD, 48, 48, 8, 2, 1, 1)
  K(ROLE_RES_A, 48, 48, 8, 2, 1, 1)
  K(ROLE_RES_B, 48, 48, 8, 2, 1, 1)
  K(ROLE_TAIL, 48, 16, 16, 4, 2, 1)
  K(ROLE_TAIL, 48, 16, 8, 2, 3, 1)
  K(ROLE_TAIL, 48, 16, 8, 2, 4, 1)
  K(ROLE_TINY0, 48, 48, 8, 2, 1, 1)
  K(ROLE_UP, 48, 32, 16, 4, 1, 2)
  K(ROLE_UP, 48, 32, 8, 2, 2, 2)
  K(ROLE_UP, 48, 48, 8, 2, 1, 3)
  K(ROLE_BODY, 64, 64, 8, 2, 1, 1)
  K(ROLE_HEAD, 64, 64, 8, 2, 1, 1)
  K(ROLE_RES_A, 64, 64, 8, 2, 1, 1)
  K(ROLE_RES_B, 64, 64, 8, 2, 1, 1)
  K(ROLE_TAIL, 64, 16, 16, 2, 2, 1)
  K(ROLE_TAIL, 64, 16, 8, 2, 3, 1)
  K(ROLE_TAIL, 64, 16, 8, 1, 4, 1)
  K(ROLE_TINY0, 64, 64, 8, 2, 1, 1)
  K(ROLE_UP, 64, 48, 8, 2, 1, 3)
  K(ROLE_UP, 64, 64, 8, 2, 1, 2)
  K(ROLE_UP, 64, 64, 4, 1, 2, 2)
  K(ROLE_FOLD, 16, 80, 4, 1, 1, 1)
  K(ROLE_FOLD, 16, 48, 8, 2, 1, 1)
  K(ROLE_FOLD, 16, 48, 4, 1, 2, 1)
  K(ROLE_FOLD, 32, 80, 4, 1, 1, 1)
  K(ROLE_FOLD, 32, 48, 8, 2, 1, 1)
  K(ROLE_FOLD, 32, 48, 4, 1, 2, 1)
  K(ROLE_FOLD, 48, 80, 4, 1, 1, 1)
  K(ROLE_FOLD, 48, 48, 8, 2, 1, 1)
  K(ROLE_FOLD, 48, 48, 4, 1, 2, 1)
  K(ROLE_FOLD, 64, 80, 4, 1, 1, 1)
  K(ROLE_FOLD, 64, 48, 8, 2, 1, 1)
  K(ROLE_FOLD, 64, 48, 4, 1, 2, 1)
  K(ROLE_FOLDF, 16, 80, 6, 1, 1, 3)
  K(ROLE_FOLDF, 16, 48, 6, 1, 1, 2)
  K(ROLE_FOLDF, 32, 80, 6, 1, 1, 3)
  K(ROLE_FOLDF, 32, 48, 6, 1, 1, 2)
  K(ROLE_FOLDF, 48, 80, 6, 1, 1, 3)
  K(ROLE_FOLDF, 48, 48, 6, 1, 1, 2)
  K(ROLE_FOLDF, 64, 80, 6, 1, 1, 3)
  K(ROLE_FOLDF, 64, 48, 6, 1, 1, 2)
#undef K
  return nullptr;
}

}  // namespace tc

// Repack the (bf16-rounded) weights into per-conv tcgen05 B images.
regen_status conv_tc_prepare(SRNet* net) {
  using namespace tc;
  net->use_tc = false;
  if (net->cfg.dtype != REGEN_DTYPE_BF16 || net->cfg.channels % 16 != 0) return REGEN_OK;
  const char* force = getenv("REGEN_FORCE_SIMT");   // debugging aid: run every conv on the SIMT kernel
  if (force && force[0] == '1') return REGEN_OK;
  size_t total = 0;
  for (auto& d : net->convs) total = std::max(total, d.b_off + (size_t)d.cout);
  std::vector<float> w32(total);
  cudaError_t e = cudaMemcpy(w32.data(), net->d_w32, total * sizeof(float), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    set_error("weights readback: %s", cudaGetErrorString(e));
    return REGEN_E_CUDA;
  }
  net->tc_plans = new NetPlans();
  net->use_tc = true;
  net->tc_weights.assign(w32.begin(), w32.end());   // kept for bin-width dependent planning
  return REGEN_OK;
}

void conv_tc_release(SRNet* net) {
  delete (tc::NetPlans*)net->tc_plans;
  net->tc_plans = nullptr;
}

// Every conv's plan and B image for the handle's bin width are built once, by regen_sr_create
// (conv_tc_plan_all); launches only read them (the handle is immutable afterwards).
regen_status conv_tc_plan_all(SRNet* net, int bin_w) {
  using namespace tc;
  NetPlans* np = (NetPlans*)net->tc_plans;
  REGEN_REQUIRE(np != nullptr, "tcgen05 weights not prepared");
  np->plans.assign(net->convs.size(), Plan());
  net->tc_bin_w = bin_w;
  std::vector<uint8_t> all;
  for (size_t i = 0; i < net->convs.size(); ++i) {
    ConvDesc& d = net->convs[i];
    std::vector<float> W((size_t)d.cout * d.cin * 9);
    for (int co = 0; co < d.cout; ++co)
      for (int ci = 0; ci < d.cin; ++ci)
        for (int t = 0; t < 9; ++t)
          W[((size_t)co * d.cin + ci) * 9 + t] = net->tc_weights[d.w_off + ((size_t)co * d.cin8 * 8 + ci) * 9 + t];
    Plan q;
    std::vector<uint16_t> img;
    if (plan_conv(d, net->cfg.channels, d.res, bin_w, q, img, W.data()) &&
        lookup(d.role, net->cfg.channels, q.cp, q.R, q.G, q.T, d.ps) != nullptr) {
      all.resize((all.size() + 1023) / 1024 * 1024);
      d.tc_off = all.size();
      const uint8_t* bb = reinterpret_cast<const uint8_t*>(img.data());
      all.insert(all.end(), bb, bb + img.size() * 2);
      np->plans[i] = q;
    } else {
      np->plans[i].cp = -1;
    }
  }
  cudaFree(net->d_wtc);
  net->d_wtc = nullptr;
  if (!all.empty()) {
    REGEN_CUDA(cudaMalloc(&net->d_wtc, all.size()));
    REGEN_CUDA(cudaMemcpy(net->d_wtc, all.data(), all.size(), cudaMemcpyHostToDevice));
  }
  net->wtc_bytes = all.size();
  return REGEN_OK;
}

static const tc::Plan* tc_plan_of(const SRNet* net, const ConvDesc& cv, int bin_w) {
  const tc::NetPlans* np = (const tc::NetPlans*)net->tc_plans;
  if (np == nullptr || net->tc_bin_w != bin_w || np->plans.size() != net->convs.size()) return nullptr;
  const tc::Plan& q = np->plans[&cv - net->convs.data()];
  return q.ok ? &q : nullptr;
}

bool conv_tc_supported(const SRNet* net, const ConvDesc& cv, int bin_w) {
  if (!net->use_tc) return false;
  return tc_plan_of(net, cv, bin_w) != nullptr;
}

regen_status conv_tc_launch(const SRNet* net, const ConvDesc& cv, const void* in, void* out, const void* skip,
                            const uint32_t* mbits, int max_bins, const int32_t* d_num_bins, int bin_w, int bin_h,
                            int* counter, cudaStream_t s, int reverse) {
  using namespace tc;
  const Plan* pl = tc_plan_of(net, cv, bin_w);
  REGEN_REQUIRE(pl != nullptr, "no tcgen05 plan for conv");
  Params p;
  memset(&p, 0, sizeof(p));
  p.in = (const __nv_bfloat16*)in;
  p.out = (__nv_bfloat16*)out;
  p.skip = (const __nv_bfloat16*)skip;
  p.bias = net->d_w32 + cv.b_off;
  p.mbits = mbits;
  p.num_bins = d_num_bins;
  p.wimg = net->d_wtc + cv.tc_off;
  p.b_bytes = pl->b_bytes;
  p.Wr = bin_w * cv.res;
  p.Hr = bin_h * cv.res;
  p.res = cv.res;
  p.bin_w = bin_w;
  p.bin_h = bin_h;
  p.cout = cv.cout;
  p.nchunk = pl->nchunk;
  p.nbands = (p.Hr + BR - 1) / BR;
  p.max_bins = max_bins;
  p.out_c8 = cv.role == ROLE_UP ? net->cfg.channels / 8 : (cv.cout + 7) / 8;
  p.res_scale = cv.role == ROLE_RES_B ? net->cfg.res_scale : 1.0f;
  p.counter = counter;
  p.reverse = reverse;
  const int cin8 = cv.cin == 3 ? 1 : cv.cin / 8;
  const uint32_t grp_bytes = (uint32_t)cin8 * p.Wr * 16 * pl->G;
  // deepest input ring that fits (row loads are latency-bound: more rows in flight per SM)
  const size_t bbytes_all = (size_t)pl->b_bytes * (pl->nchunk > 1 ? 2 : 1);
  int gslog = 3;
  while (gslog > 0 && 1024 + ((size_t)1 << gslog) * grp_bytes + bbytes_all > 220 * 1024) --gslog;
  p.ngs = 1 << gslog;
  p.gslog = gslog;
  const size_t smem = 1024 + (size_t)p.ngs * grp_bytes + bbytes_all;
  REGEN_REQUIRE(smem <= 227 * 1024, "conv SMEM %zu too large", smem);
  KernFn kern = lookup(cv.role, net->cfg.channels, pl->cp, pl->R, pl->G, pl->T, cv.ps);
  REGEN_REQUIRE(kern != nullptr, "no tcgen05 kernel instance");
  REGEN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nsm = net->n_sm;
  const int units = max_bins * p.nbands * pl->nchunk;
  const int grid = std::min(units, nsm);
  static unsigned long long* d_prof = nullptr;
  static int prof_on = -1;
  if (prof_on < 0) {
    const char* e = getenv("REGEN_TC_PROF");
    prof_on = (e && e[0] == '1') ? 1 : 0;
    if (prof_on) cudaMalloc(&d_prof, 16 * sizeof(unsigned long long));
  }
  if (prof_on) {
    cudaMemsetAsync(d_prof, 0, 16 * sizeof(unsigned long long), s);
    p.prof = d_prof;
  }
  static const char* kRoleName[] = {"conv_head", "conv_res_a", "conv_res_b", "conv_body", "conv_up", "conv_tail",
                                    "conv_tiny0", "conv_tiny1", "conv_fold"};
  REGEN_TRACE(kRoleName[cv.role], s);
  kern<<<grid, NTHREADS, smem, s>>>(p);
  REGEN_LAUNCH_CHECK();
  if (prof_on) {
    unsigned long long h[8];
    cudaMemcpyAsync(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double g = (double)grid;
    fprintf(stderr,
            "[tc-prof] role=%d CP=%d R=%d G=%d T=%d chunks=%d gslots=%d | producer total %.0f wait_empty %.0f | "
            "mma total %.0f waits %.0f | epi total %.0f wait_accfull %.0f rearm %.0f (cycles/CTA)\n",
            cv.role, pl->cp, pl->R, pl->G, pl->T, pl->nchunk, p.ngs, h[4] / g, h[0] / g, h[5] / g, h[1] / g,
            h[6] / (8 * g), h[3] / (8 * g), h[7] / (8 * g));
  }
  return REGEN_OK;
}

}  // namespace regen

// ---------------------------------------------------------------------------------- fused fold
// The fold conv (ROLE_FOLD's B image and bias) run as ROLE_FOLDF: bands of 64 rows (66 computed),
// a 6-slot TMEM ring, and 4 combiner warps that turn the partial sums into the owned MBs' HR pixels.
namespace regen {

static const tc::Plan* foldf_plan(const SRNet* net, int bin_w, int& ps) {
  if (!net->use_tc || net->fold_conv < 0) return nullptr;
  const ConvDesc& cv = net->convs[net->fold_conv];
  const tc::Plan* pl = tc_plan_of(net, cv, bin_w);
  if (pl == nullptr || pl->T != 1 || cv.res != 1 || pl->nchunk != 1) return nullptr;
  ps = net->convs[net->fold_conv - 2].ps;
  if (tc::lookup(ROLE_FOLDF, net->cfg.channels, pl->cp, 6, 1, 1, ps) == nullptr) return nullptr;
  // SMEM with the shallowest input ring (2 rows): guard + rows + B image + partial-sum rows
  const size_t need = 1024 + 2ull * (cv.cin / 8) * bin_w * 16 + pl->b_bytes + (size_t)tc::FF_NPR * (pl->cp / 8) * tc::FF_W * 16;
  if (need > 224 * 1024) return nullptr;
  return pl;
}

bool fold_fused_supported(const SRNet* net, int bin_w) {
  int ps = 0;
  if (net->no_foldf) return false;   // REGEN_NO_FOLDF=1 at create: the fold conv + standalone combine (A/B aid)
  return foldf_plan(net, bin_w, ps) != nullptr;
}

regen_status fold_fused_launch(const SRNet* net, const void* in, const uint32_t* mbits, int max_bins,
                               const int32_t* d_num_bins, int bin_w, int bin_h, int* counter, cudaStream_t s,
                               int reverse, const FoldFrameArgs& fa) {
  using namespace tc;
  int ps = 0;
  const Plan* pl = foldf_plan(net, bin_w, ps);
  REGEN_REQUIRE(pl != nullptr, "no fused fold plan");
  const ConvDesc& cv = net->convs[net->fold_conv];
  const ConvDesc& tail = net->convs[net->fold_conv - 1];
  Params p;
  memset(&p, 0, sizeof(p));
  p.in = (const __nv_bfloat16*)in;
  p.bias = net->d_w32 + cv.b_off;
  p.mbits = mbits;
  p.num_bins = d_num_bins;
  p.wimg = net->d_wtc + cv.tc_off;
  p.b_bytes = pl->b_bytes;
  p.Wr = bin_w;
  p.Hr = bin_h;
  p.res = 1;
  p.bin_w = bin_w;
  p.bin_h = bin_h;
  p.cout = cv.cout;
  p.nchunk = 1;
  p.nbands = (bin_h + 63) / 64;
  p.max_bins = max_bins;
  p.out_c8 = (cv.cout + 7) / 8;
  p.res_scale = 1.0f;
  p.counter = counter;
  p.reverse = reverse;
  p.fdst = fa.dst;
  p.fout = fa.out;
  p.tbias = net->d_w32 + tail.b_off;
  p.fout_mode = fa.out_dtype;
  p.fOW = fa.geom.frame_w * net->cfg.scale;
  {
    const char* e = getenv("REGEN_FF_DEBUG");
    p.ff_debug = e ? atoi(e) : 0;
  }
  const uint32_t grp_bytes = (uint32_t)(cv.cin / 8) * p.Wr * 16;   // G = 1
  // ring depths: the deepest partial-sum ring (the epilogue and the combines decoupled) that leaves
  // room for >= 4 input rows in flight, else the shallowest
  const size_t prow = (size_t)(pl->cp / 8) * FF_W * 16;
  p.npr = FF_NPR;
  for (int n = FF_NPR_MAX; n > FF_NPR; --n)
    if (1024 + 4ull * grp_bytes + pl->b_bytes + n * prow <= 224 * 1024) { p.npr = n; break; }
  if (const char* e = getenv("REGEN_FF_NPR")) p.npr = std::max(FF_NPR, std::min(FF_NPR_MAX, atoi(e)));   // A/B aid
  const size_t pring = (size_t)p.npr * prow;
  int gslog = 3;
  while (gslog > 1 && 1024 + ((size_t)1 << gslog) * grp_bytes + pl->b_bytes + pring > 224 * 1024) --gslog;
  p.ngs = 1 << gslog;
  p.gslog = gslog;
  const size_t smem = 1024 + (size_t)p.ngs * grp_bytes + pl->b_bytes + pring;
  REGEN_REQUIRE(smem <= 227 * 1024, "fused fold SMEM %zu too large", smem);
  KernFn kern = lookup(ROLE_FOLDF, net->cfg.channels, pl->cp, 6, 1, 1, ps);
  REGEN_REQUIRE(kern != nullptr, "no fused fold kernel instance");
  REGEN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::min(max_bins * p.nbands, net->n_sm);
  static unsigned long long* d_prof = nullptr;
  static int prof_on = -1;
  if (prof_on < 0) {
    const char* e = getenv("REGEN_TC_PROF");
    prof_on = (e && e[0] == '1') ? 1 : 0;
    if (prof_on) cudaMalloc(&d_prof, 16 * sizeof(unsigned long long));
  }
  if (prof_on) {
    cudaMemsetAsync(d_prof, 0, 16 * sizeof(unsigned long long), s);
    p.prof = d_prof;
  }
  REGEN_TRACE("conv_fold_frames", s);
  kern<<<grid, NTHREADS + 256, smem, s>>>(p);
  REGEN_LAUNCH_CHECK();
  if (prof_on) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double g = (double)grid;
    fprintf(stderr,
            "[tc-prof] fused fold CP=%d gslots=%d | producer total %.0f wait_empty %.0f | mma total %.0f wait_accempty %.0f "
            "wait_infull %.0f | "
            "epi total %.0f wait_accfull %.0f rearm %.0f wait_ring %.0f | combine total %.0f wait_rows %.0f "
            "(cycles/CTA, per warp)\n",
            pl->cp, p.ngs, h[4] / g, h[0] / g, h[5] / g, h[1] / g, h[2] / g, h[6] / (8 * g), h[3] / (8 * g), h[7] / (8 * g),
            h[8] / (8 * g), h[10] / (8 * g), h[9] / (8 * g));
  }
  return REGEN_OK;
}

}  // namespace regen
