// Fused EDSR residual block on tcgen05 (sm_100a): r' = mask * (r + res_scale * conv_b(relu(conv_a(r))))
// with the intermediate t = mask * relu(conv_a(r)) kept in SMEM (reading D8/D11 of DESIGN.md).
//
// Both convs use the sliding-window mapping of conv_tc.cu (kernel rows folded into N = 3*C, one MMA
// per (dx, K-chunk pair) per input row, output-row accumulators in a TMEM ring at decreasing
// columns). A work unit is a band of BR = 32 output rows of one bin:
//   conv_a reads r rows y0-2 .. y1+1 (36 rows, bulk-copied in groups of G = 1 row) and produces t rows
//   y0-1 .. y1 (34 rows) into TMEM ring A; the quad-A epilogue warps (warps 2-9: two groups of four
//   taking alternate rows) apply bias/ReLU/mask and write each t row into an SMEM ring in the UMMA
//   operand layout (generic-proxy stores + proxy fence); conv_b consumes those t rows from SMEM into
//   TMEM ring B; the quad-B warps (10-17) add the residual r and store r'. The residual rows are
//   bulk-copied into their own SMEM ring by warp 19 (an L2 re-read of rows the producer loaded a few
//   rows earlier), so no global-load latency sits on the epilogue's path; the occupancy words of a
//   unit's rows are fetched once per unit. Each epilogue releases its accumulator slot (TMEM loads,
//   re-arm) before it waits for its t-ring / store slot.
// Two issuing threads: warp 1 issues conv_a, warp 18 conv_b (each waits only on its own inputs).
// Synchronisation is per group of G rows: r ring (in_full/in_empty), TMEM ring A and B
// (acc*_full/acc*_empty), t ring (t_full by quad A, t_empty by tcgen05.commit), residual ring
// (res_full by the bulk copy, res_empty by quad B).
// TMEM rings: R logical slots plus GU = 2 guard slots (see RShape); every unit starts at an
// accumulator sequence that is a multiple of R (the group count per unit is padded with empty
// "phantom" groups that only cycle the barriers), so a row's TMEM columns, and the split of its sum
// between slot and guard, depend on its band-local index only: results do not depend on which CTA
// computed a unit, and every TMEM column in the MMA stream is a compile-time constant.
// HBM traffic per block: read r (+ its L2-hot re-read as the residual) and write r' once, instead
// of r, t, t, r, r' for two separate convs.
#include <stdlib.h>

#include <vector>

#include "tc_common.cuh"

namespace regen {
namespace tc {

namespace rb {

// warp 0 r-row producer, 1 conv_a MMAs, 2 .. 2+8*EPG-1 epilogues (quad A then quad B, each EPG groups of
// 4 warps taking alternate accumulator groups), then the conv_b MMA warp and the residual-row producer
constexpr int EPG = 2;
constexpr int NEPI = 8 * EPG;              // epilogue warps
constexpr int W_MMAB = 2 + NEPI, W_RES = 3 + NEPI;
constexpr int NTHREADS = 32 * (4 + NEPI);
constexpr int BR = 32;        // output rows per unit
constexpr int NA_OUT = BR + 2;   // t rows per unit
constexpr int NA_IN = BR + 4;    // r rows per unit

struct Params {
  const __nv_bfloat16* in;    // r
  __nv_bfloat16* out;         // r'
  const float* bias_a;
  const float* bias_b;
  const uint32_t* mbits;
  const int32_t* num_bins;
  const uint8_t* wimg;        // [B image conv_a][B image conv_b]
  uint32_t b_bytes;           // bytes of one image
  int Hr, bin_w, bin_h, max_bins, nbands;
  float res_scale;
  int* counter;
  unsigned long long* prof;   // REGEN_TC_PROF=1: wait-time counters
  int reverse;                // hand out units last-to-first (L2 reuse along the chain)
  int dbg;                    // REGEN_RB_DBG bits (timing experiments only): 1 no epilogue work, 2 no row loads, 4 no MMAs,
                              // 8 no TMEM loads, 16 no TMEM re-arm stores, 32 no t-row / r' stores, 64 no proxy fence,
                              // 128 no r' stores, 256 no t-row stores
};

// R logical accumulator slots per ring plus GU guard slots (0 or 2) after them: with guards the 3-row
// window that starts at slot s0 >= R-2 runs on into the guards instead of wrapping to slot 0, so every
// row issues one N = 3C MMA per step (no 2-MMA split re-reading the A tile); a row at logical slot
// s < GU then holds part of its sum in guard R+s, which its epilogue adds and re-arms with zero.
template <int C, int R, int G, int GU>
struct RShape {
  static constexpr int KC = C / 16, NS = 3 * KC, N = 3 * C;
  static constexpr int RP = R + GU;                      // physical slots per ring
  static constexpr int NSLOT = G * C <= 32 ? 8 : 4;      // r-ring and t-ring groups (power of two)
  static constexpr int NGA_IN = (NA_IN + G - 1) / G;
  static constexpr int NGA_OUT = (NA_OUT + G - 1) / G;   // = t groups = conv_b input groups
  static constexpr int NGB_OUT = BR / G;
  static constexpr int OGR = R / G;
  static constexpr int NRES = G == 1 ? 6 : 3;            // residual-ring groups
  static constexpr int NGA_PAD = (NGA_OUT + OGR - 1) / OGR * OGR;   // + phantom groups
  static constexpr int NGB_PAD = (NGB_OUT + OGR - 1) / OGR * OGR;
  static constexpr int COLB = RP * C;                    // TMEM column of ring B
  static_assert(2 * RP * C <= 512 && R % G == 0 && OGR >= 3 && BR % G == 0 && OGR <= 16, "shape");
  static_assert(GU == 0 || GU == 2, "guards");
  // input group whose processing completes accumulator group k of a conv with NOUT real rows
  __host__ __device__ static constexpr int done_group(int k, int nout) {
    return ((G * k + G - 1 < nout ? G * k + G - 1 : nout - 1) + 2) / G;
  }
};

// TMEM slot of band-local output row j (every unit starts at a sequence that is a multiple of R)
template <int R>
__host__ __device__ constexpr uint32_t ring_slot(int j) { return (uint32_t)((R - j % R) % R); }

// Issue the sliding-window MMAs of one input row: `i` = unit-local input row, `nout` = number of real
// output rows, `tmem` = TMEM column of the ring, `a_row16` = the row's SMEM address (16-B units),
// `b16` = B image base (16-B units). Every column is a compile-time constant after unrolling.
template <int C, int R, int G, int GU>
__device__ __forceinline__ void issue_row(int i, int nout, uint32_t tmem, uint32_t a_row16, uint32_t b16,
                                         uint32_t en) {
  using S = RShape<C, R, G, GU>;
  constexpr uint32_t BLBO = (uint32_t)S::N;
  const int gA = i < nout ? 0 : (i - 1 < nout ? 1 : 2);
  const int gB = i >= 2 ? 3 : (i >= 1 ? 2 : 1);
  if (gA >= gB) return;   // compile-time after unrolling
  const uint32_t ng = (uint32_t)(gB - gA);
  const uint32_t s0 = ring_slot<R>(i - gA);
  const uint32_t len1 = GU ? ng : min(ng, (uint32_t)R - s0);   // guards: never split
  const uint32_t two = (len1 < ng && en) ? 1u : 0u;
  const uint32_t idesc1 = make_idesc((int)(len1 * C)), idesc2 = make_idesc((int)((ng - len1) * C));
  const uint32_t d1 = tmem + s0 * (uint32_t)C;
#pragma unroll
  for (int st = 0; st < S::NS; ++st) {
    const int dx = st / S::KC - 1, plane = 2 * (st % S::KC);
    const uint32_t a_lo = (a_row16 + (uint32_t)(plane * 128) + (uint32_t)dx) + (128u << 16);   // LBO = plane
    const uint32_t b_lo = (b16 + (uint32_t)(st * S::N * 2) + (uint32_t)(gA * C)) + (BLBO << 16);
    mma_bf16(d1, a_lo, b_lo, idesc1, en);
    if (!GU) mma_bf16(tmem, a_lo, b_lo + len1 * (uint32_t)C, idesc2, two);
  }
}

// an accumulator row (C fp32 columns) into registers; a row with part of its sum in a guard slot
// (warp-uniform `guarded`) adds the guard's columns
template <int C, int GU>
__device__ __forceinline__ void load_row(uint32_t taddr, uint32_t gaddr, bool guarded, uint32_t (&r)[C]) {
  if constexpr (C % 32 == 0) {
#pragma unroll
    for (int c = 0; c < C; c += 32) tmem_ld32(taddr + (uint32_t)c, r + c);
  } else {
#pragma unroll
    for (int c = 0; c < C; c += 16) tmem_ld16(taddr + (uint32_t)c, r + c);
  }
  tmem_ld_wait();
  if (GU > 0 && guarded) {   // 16 guard columns at a time (register pressure)
#pragma unroll
    for (int c = 0; c < C; c += 16) {
      uint32_t g[16];
      tmem_ld16(gaddr + (uint32_t)c, g);
      tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 16; ++e) r[c + e] = __float_as_uint(__uint_as_float(r[c + e]) + __uint_as_float(g[e]));
    }
  }
}
template <int C>
__device__ __forceinline__ void rearm_zero(uint32_t gaddr) {
  float z[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) z[e] = 0.f;
#pragma unroll
  for (int c = 0; c < C; c += 16) tmem_st16(gaddr + (uint32_t)c, z);
}

template <int C, int R, int G, int GU>
__global__ void __launch_bounds__(NTHREADS, 1) resblock_tc_kernel(const __grid_constant__ Params p) {
  using S = RShape<C, R, G, GU>;
  constexpr int NSLOT = S::NSLOT, NRES = S::NRES;
  constexpr int ROW_BYTES = (C / 8) * 128 * 16;
  constexpr int GRP = G * ROW_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t in_full[NSLOT], in_empty[NSLOT], t_full[NSLOT], t_empty[NSLOT];
  __shared__ __align__(8) uint64_t a_full[16], a_empty[16], b_fullacc[16], b_emptyacc[16];
  __shared__ __align__(8) uint64_t res_full[NRES], res_empty[NRES];
  __shared__ __align__(8) uint64_t w_full;
  __shared__ __align__(8) uint64_t unit_full[4], unit_empty[4];
  __shared__ int unit_ring[4];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(16) float bias_sm[2][64];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* rring = smem_raw + 1024;
  uint8_t* tring = rring + NSLOT * GRP;
  uint8_t* wimg = tring + NSLOT * GRP;
  uint8_t* resring = wimg + 2 * p.b_bytes;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&in_full[i], 1); mbar_init(&in_empty[i], 1);
      mbar_init(&t_full[i], 4); mbar_init(&t_empty[i], 1);
    }
    for (int i = 0; i < S::OGR; ++i) {
      mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 4);
      mbar_init(&b_fullacc[i], 1); mbar_init(&b_emptyacc[i], 4);
    }
    for (int i = 0; i < NRES; ++i) { mbar_init(&res_full[i], 1); mbar_init(&res_empty[i], 4); }
    mbar_init(&w_full, 1);
    for (int i = 0; i < 4; ++i) { mbar_init(&unit_full[i], 1); mbar_init(&unit_empty[i], 3 + NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int n = threadIdx.x; n < 64; n += NTHREADS) {
    bias_sm[0][n] = n < C ? __ldg(p.bias_a + n) : 0.f;
    bias_sm[1][n] = n < C ? __ldg(p.bias_b + n) : 0.f;
  }
  // zero the t ring (rows read at the left/right halo of masked pixels must be finite)
  for (int i = threadIdx.x; i < NSLOT * GRP / 16; i += NTHREADS) reinterpret_cast<uint4*>(tring)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  // arm both accumulator rings with their biases (guard slots with zero)
  if (warp >= 2 && warp < 2 + NEPI && ((warp - 2) >> 2) % EPG == 0) {
    const int quad = (warp - 2) >> 2 >= EPG ? 1 : 0, q4 = warp & 3;
    float z[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) z[e] = 0.f;
    for (int s = 0; s < S::RP; ++s)
#pragma unroll
      for (int c0 = 0; c0 < C; c0 += 16)
        tmem_st16(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)(quad * S::COLB + s * C + c0),
                  s < R ? bias_sm[quad] + c0 : z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int nbins = min(*p.num_bins, p.max_bins);
  const int total_units = nbins * p.nbands;
  uint32_t w_ae = 0, w_if = 0, w_be = 0, w_tf = 0, w_ea = 0, w_te = 0, w_eb = 0, w_rs = 0;
  const long long pstart = clock64();

  if (warp == 0) {
    // =============================== producer: r rows ===============================
    if (lane == 0) {
      mbar_expect_tx(&w_full, 2 * p.b_bytes);
      bulk_g2s(wimg, p.wimg, 2 * p.b_bytes, &w_full);
      uint32_t ig = 0;
      for (uint32_t us = 0;; ++us) {
        int u = atomicAdd(p.counter, 1);
        if (u >= total_units) u = -1;
        else if (p.reverse) u = total_units - 1 - u;
        mbar_wait(&unit_empty[us & 3], ((us >> 2) & 1) ^ 1);
        unit_ring[us & 3] = u;
        mbar_arrive(&unit_full[us & 3]);
        if (u < 0) break;
        const int bin = u / p.nbands, y0 = (u - bin * p.nbands) * BR;
        const int y1 = min(p.Hr, y0 + BR);
        const int rlo = max(y0 - 2, 0), rhi = min(y1 + 1, p.Hr - 1);
        for (int k = 0; k < S::NGA_IN; ++k, ++ig) {
          const uint32_t slot = ig & (NSLOT - 1);
          mbar_wait(&in_empty[slot], ((ig / NSLOT) & 1) ^ 1);
          const int g0 = y0 - 2 + G * k;
          const int a = max(g0, rlo), b = min(g0 + G - 1, rhi);
          if (a <= b && !(p.dbg & 2)) {
            mbar_expect_tx(&in_full[slot], (uint32_t)(b - a + 1) * ROW_BYTES);
            bulk_g2s(rring + slot * GRP + (uint32_t)(a - g0) * ROW_BYTES,
                     p.in + ((size_t)bin * p.Hr + a) * (ROW_BYTES / 2), (uint32_t)(b - a + 1) * ROW_BYTES,
                     &in_full[slot]);
          } else {
            mbar_arrive(&in_full[slot]);
          }
        }
      }
    }
  } else if (warp == W_RES) {
    // =============================== producer: residual rows (quad B's r) ===============================
    if (lane == 0) {
      uint32_t rs = 0;
      for (uint32_t us = 0;; ++us) {
        mbar_wait(&unit_full[us & 3], (us >> 2) & 1);
        const int u = *(volatile int*)&unit_ring[us & 3];
        mbar_arrive(&unit_empty[us & 3]);
        if (u < 0) break;
        const int bin = u / p.nbands, y0 = (u - bin * p.nbands) * BR;
        const int nrows = min(BR, p.Hr - y0);
        for (int jb = 0; jb < S::NGB_OUT; ++jb, ++rs) {
          const uint32_t slot = rs % NRES;
          mbar_wait(&res_empty[slot], ((rs / NRES) & 1) ^ 1);
          const int a = G * jb, n = min(G, nrows - a);
          if (n > 0 && !(p.dbg & 1)) {
            mbar_expect_tx(&res_full[slot], (uint32_t)n * ROW_BYTES);
            bulk_g2s(resring + slot * GRP, p.in + ((size_t)bin * p.Hr + y0 + a) * (ROW_BYTES / 2),
                     (uint32_t)n * ROW_BYTES, &res_full[slot]);
          } else {
            mbar_arrive(&res_full[slot]);
          }
        }
      }
    }
  } else if (warp == 1 || warp == W_MMAB) {
    // =============================== MMA issuers: conv_a (warp 1), conv_b (warp 10) ===============
    // Two issuing threads, so a conv_b wait for a t row never holds back conv_a's MMAs (tcgen05.commit
    // tracks the MMAs of the committing thread only).
    if (elect_one()) {
      const bool conv_a = warp == 1;
      uint32_t ig = 0, tg = 0;      // r-ring groups consumed, t-ring groups consumed
      uint32_t qa = 0, qb = 0;      // accumulator group sequences (ring A, ring B; multiples of OGR per unit)
      const uint32_t r16 = smem_u32(rring) >> 4, t16 = smem_u32(tring) >> 4;
      const uint32_t ba16 = smem_u32(wimg) >> 4, bb16 = (smem_u32(wimg) + p.b_bytes) >> 4;
      mbar_wait(&w_full, 0);
      for (uint32_t us = 0;; ++us) {
        mbar_wait(&unit_full[us & 3], (us >> 2) & 1);
        const int u = *(volatile int*)&unit_ring[us & 3];
        mbar_arrive(&unit_empty[us & 3]);
        if (u < 0) break;
        const int bin = u / p.nbands, y0 = (u - bin * p.nbands) * BR;
        const int y1 = min(p.Hr, y0 + BR);
        const int rlo = max(y0 - 2, 0), rhi = min(y1 + 1, p.Hr - 1);
        if (conv_a) {
#pragma unroll
          for (int k = 0; k < S::NGA_IN; ++k) {
            // ---- conv_a, input group k: r rows y0-2 + G*k ...
            const uint32_t slot = (ig + k) & (NSLOT - 1);
            if (k < S::NGA_OUT) { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&a_empty[(qa + k) % S::OGR], (((qa + k) / S::OGR) & 1) ^ 1); if (p.prof) w_ae += (uint32_t)clock() - t0_; }
            { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&in_full[slot], ((ig + k) / NSLOT) & 1); if (p.prof) w_if += (uint32_t)clock() - t0_; }
            tc_fence_after();
#pragma unroll
            for (int ii = 0; ii < G; ++ii) {
              const int i = G * k + ii;
              if (i >= NA_IN) continue;
              const int r = y0 - 2 + i;
              const uint32_t en = (r >= rlo && r <= rhi && !(p.dbg & 4)) ? 1u : 0u;
              issue_row<C, R, G, GU>(i, NA_OUT, tmem, r16 + slot * (GRP / 16) + ii * (ROW_BYTES / 16), ba16, en);
            }
            mma_commit(&in_empty[slot]);
#pragma unroll
            for (int ka = 0; ka < S::NGA_OUT; ++ka)
              if (S::done_group(ka, NA_OUT) == k) mma_commit(&a_full[(qa + ka) % S::OGR]);
            if (k == S::NGA_IN - 1) {   // groups whose completion falls past the last input group
#pragma unroll
              for (int ka = 0; ka < S::NGA_OUT; ++ka)
                if (S::done_group(ka, NA_OUT) > k) mma_commit(&a_full[(qa + ka) % S::OGR]);
            }
          }
#pragma unroll
          for (int ka = S::NGA_OUT; ka < S::NGA_PAD; ++ka) {   // phantom groups: cycle the barriers only
            mbar_wait(&a_empty[(qa + ka) % S::OGR], (((qa + ka) / S::OGR) & 1) ^ 1);
            mma_commit(&a_full[(qa + ka) % S::OGR]);
          }
        } else {
#pragma unroll
          for (int kb = 0; kb < S::NGA_OUT; ++kb) {
            // ---- conv_b, input group kb: t rows y0-1 + G*kb ... (SMEM t ring)
            const uint32_t tslot = (tg + kb) & (NSLOT - 1);
            if (kb < S::NGB_OUT) { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&b_emptyacc[(qb + kb) % S::OGR], (((qb + kb) / S::OGR) & 1) ^ 1); if (p.prof) w_be += (uint32_t)clock() - t0_; }
            { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&t_full[tslot], ((tg + kb) / NSLOT) & 1); if (p.prof) w_tf += (uint32_t)clock() - t0_; }
            tc_fence_after();
#pragma unroll
            for (int ii = 0; ii < G; ++ii) {
              const int i = G * kb + ii;
              if (i >= NA_OUT) continue;
              const int tr = y0 - 1 + i;
              const uint32_t en = (tr >= 0 && tr < p.Hr && !(p.dbg & 4)) ? 1u : 0u;
              issue_row<C, R, G, GU>(i, BR, tmem + S::COLB, t16 + tslot * (GRP / 16) + ii * (ROW_BYTES / 16), bb16, en);
            }
            mma_commit(&t_empty[tslot]);
#pragma unroll
            for (int jb = 0; jb < S::NGB_OUT; ++jb)
              if (S::done_group(jb, BR) == kb) mma_commit(&b_fullacc[(qb + jb) % S::OGR]);
            if (kb == S::NGA_OUT - 1) {
#pragma unroll
              for (int jb = 0; jb < S::NGB_OUT; ++jb)
                if (S::done_group(jb, BR) > kb) mma_commit(&b_fullacc[(qb + jb) % S::OGR]);
            }
          }
#pragma unroll
          for (int jb = S::NGB_OUT; jb < S::NGB_PAD; ++jb) {   // phantom groups
            mbar_wait(&b_emptyacc[(qb + jb) % S::OGR], (((qb + jb) / S::OGR) & 1) ^ 1);
            mma_commit(&b_fullacc[(qb + jb) % S::OGR]);
          }
        }
        ig += S::NGA_IN;
        tg += S::NGA_OUT;
        qa += S::NGA_PAD;
        qb += S::NGB_PAD;
      }
    }
    __syncwarp();
  } else {
    // =============================== epilogues ===============================
    const int egrp = (warp - 2) >> 2;
    const int quad = egrp >= EPG ? 1 : 0;    // 0: t = relu(conv_a) -> SMEM; 1: r' = r + s*conv_b -> HBM
    const int par = egrp % EPG;              // this group takes accumulator groups par, par + EPG, ...
    const int q4 = warp & 3;
    const int m = 32 * q4 + lane;
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    const int words = p.bin_w / 32;
    const size_t bin_px = (size_t)p.Hr * 128;
    constexpr size_t PSTRIDE = 128 * 8;      // elements between planes of one row
    uint32_t tg = 0, qa = 0, qb = 0, rs = 0;
    for (uint32_t us = 0;; ++us) {
      mbar_wait(&unit_full[us & 3], (us >> 2) & 1);
      const int u = *(volatile int*)&unit_ring[us & 3];
      __syncwarp();
      if (lane == 0) mbar_arrive(&unit_empty[us & 3]);
      if (u < 0) break;
      const int bin = u / p.nbands, y0 = (u - bin * p.nbands) * BR;
      const int nrows = min(BR, p.Hr - y0);
      const uint32_t* mrows = p.mbits + (size_t)bin * p.bin_h * words + q4;   // this warp's 32 pixels
      if (quad == 0) {
        // ---- t rows y0-1 .. y0+32 into the SMEM t ring; occupancy words of rows ja = lane, 32 + lane
        const uint32_t occ0 = __ldg(mrows + (size_t)min(max(y0 - 1 + lane, 0), p.Hr - 1) * words);
        const uint32_t occ1 = __ldg(mrows + (size_t)min(max(y0 + 31 + (lane & 1), 0), p.Hr - 1) * words);
        for (int ka = par; ka < S::NGA_PAD; ka += EPG) {
          const uint32_t gi = (qa + ka) % S::OGR, gph = ((qa + ka) / S::OGR) & 1;
          if (ka >= S::NGA_OUT) {   // phantom group
            mbar_wait(&a_full[gi], gph);
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[gi]);
            continue;
          }
          const uint32_t tslot = (tg + ka) & (NSLOT - 1);
          { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&a_full[gi], gph); if (p.prof) w_ea += (uint32_t)clock() - t0_; }
          tc_fence_after();
          // accumulators -> bias/ReLU/mask/bf16 in registers; slots re-armed and released before the
          // t-row stores wait for their SMEM slot
          uint4 q[G][C / 8];
#pragma unroll
          for (int jj = 0; jj < G; ++jj) {
            const int ja = G * ka + jj;
            const uint32_t sl = ring_slot<R>(ja);
            const uint32_t taddr = tmem + lane_off + sl * (uint32_t)C;
            const uint32_t gaddr = tmem + lane_off + (uint32_t)(R + sl) * (uint32_t)C;   // guard (sl < GU)
            const uint32_t ow = __shfl_sync(0xffffffffu, ja < 32 ? occ0 : occ1, ja & 31);
            if (ja < NA_OUT && ow != 0u && !(p.dbg & 9)) {   // a segment with no occupied pixel is all zero
              uint32_t r[C];
              load_row<C, GU>(taddr, gaddr, GU > 0 && sl < (uint32_t)GU, r);
              const bool occ = (ow >> lane) & 1u;
#pragma unroll
              for (int g = 0; g < C / 8; ++g) {
                float v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = fmaxf(__uint_as_float(r[8 * g + e]), 0.f);
                q[jj][g] = pack8(v, occ);
              }
            } else {
#pragma unroll
              for (int g = 0; g < C / 8; ++g) q[jj][g] = make_uint4(0, 0, 0, 0);
            }
            if (!(p.dbg & 16)) {
#pragma unroll
              for (int c = 0; c < C; c += 16) tmem_st16(taddr + (uint32_t)c, bias_sm[0] + c);
              if (GU > 0 && sl < (uint32_t)GU) rearm_zero<C>(gaddr);
            }
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_empty[gi]);
          { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&t_empty[tslot], (((tg + ka) / NSLOT) & 1) ^ 1); if (p.prof) w_te += (uint32_t)clock() - t0_; }
          uint8_t* trow0 = tring + tslot * GRP;
#pragma unroll
          for (int jj = 0; jj < G; ++jj) {
            const int ja = G * ka + jj;
            if (ja < NA_OUT && !(p.dbg & 289)) {
#pragma unroll
              for (int g = 0; g < C / 8; ++g) *reinterpret_cast<uint4*>(trow0 + jj * ROW_BYTES + g * 2048 + m * 16) = q[jj][g];
            }
          }
          if (!(p.dbg & 64)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // t rows -> tensor-core reads
          __syncwarp();
          if (lane == 0) mbar_arrive(&t_full[tslot]);
        }
      } else {
        // ---- r' rows y0 .. y0+31 = r + res_scale * conv_b, masked, to HBM (r from the residual ring)
        const uint32_t occ0 = __ldg(mrows + (size_t)min(y0 + lane, p.Hr - 1) * words);
        for (int jb = par; jb < S::NGB_PAD; jb += EPG) {
          const uint32_t gi = (qb + jb) % S::OGR, gph = ((qb + jb) / S::OGR) & 1;
          if (jb >= S::NGB_OUT) {   // phantom group
            mbar_wait(&b_fullacc[gi], gph);
            __syncwarp();
            if (lane == 0) mbar_arrive(&b_emptyacc[gi]);
            continue;
          }
          const uint32_t rsq = rs + (uint32_t)jb, rslot = rsq % NRES;
          { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&res_full[rslot], (rsq / NRES) & 1); if (p.prof) w_rs += (uint32_t)clock() - t0_; }
          { const uint32_t t0_ = (uint32_t)clock(); mbar_wait(&b_fullacc[gi], gph); if (p.prof) w_eb += (uint32_t)clock() - t0_; }
          tc_fence_after();
          // accumulators + residual -> bf16 in registers; slots re-armed and released before the stores
          const uint8_t* res0 = resring + rslot * GRP + m * 16;
          uint4 q[G][C / 8];
#pragma unroll
          for (int jj = 0; jj < G; ++jj) {
            const int j = G * jb + jj;
            const uint32_t sl = ring_slot<R>(j);
            const uint32_t taddr = tmem + lane_off + (uint32_t)S::COLB + sl * (uint32_t)C;
            const uint32_t gaddr = tmem + lane_off + (uint32_t)S::COLB + (uint32_t)(R + sl) * (uint32_t)C;
            const uint32_t ow = __shfl_sync(0xffffffffu, occ0, j & 31);
            if (j < nrows && ow != 0u && !(p.dbg & 9)) {
              uint32_t r[C];
              load_row<C, GU>(taddr, gaddr, GU > 0 && sl < (uint32_t)GU, r);
              const bool occ = (ow >> lane) & 1u;
#pragma unroll
              for (int g = 0; g < C / 8; ++g) {
                const uint4 sk = *reinterpret_cast<const uint4*>(res0 + jj * ROW_BYTES + g * 2048);
                float v[8];
                const __nv_bfloat162* s2 = reinterpret_cast<const __nv_bfloat162*>(&sk);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = __bfloat1622float2(s2[e]);
                  v[2 * e] = fmaf(p.res_scale, __uint_as_float(r[8 * g + 2 * e]), f.x);
                  v[2 * e + 1] = fmaf(p.res_scale, __uint_as_float(r[8 * g + 2 * e + 1]), f.y);
                }
                q[jj][g] = pack8(v, occ);
              }
            } else {
#pragma unroll
              for (int g = 0; g < C / 8; ++g) q[jj][g] = make_uint4(0, 0, 0, 0);
            }
            if (!(p.dbg & 16)) {
#pragma unroll
              for (int c = 0; c < C; c += 16) tmem_st16(taddr + (uint32_t)c, bias_sm[1] + c);
              if (GU > 0 && sl < (uint32_t)GU) rearm_zero<C>(gaddr);
            }
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&b_emptyacc[gi]);
            mbar_arrive(&res_empty[rslot]);
          }
#pragma unroll
          for (int jj = 0; jj < G; ++jj) {
            const int j = G * jb + jj;
            if (j < nrows && !(p.dbg & 169)) {
              __nv_bfloat16* o = p.out + (size_t)bin * bin_px * C + (size_t)(y0 + j) * (C / 8) * PSTRIDE + (size_t)m * 8;
#pragma unroll
              for (int g = 0; g < C / 8; ++g) *reinterpret_cast<uint4*>(o + g * PSTRIDE) = q[jj][g];
            }
          }
        }
      }
      tg += S::NGA_OUT;
      qa += S::NGA_PAD;
      qb += S::NGB_PAD;
      rs += S::NGB_OUT;
    }
  }
  if (p.prof && lane == 0) {
    const long long tot = clock64() - pstart;
    if (warp == 1) {
      atomicAdd(p.prof + 0, (unsigned long long)tot); atomicAdd(p.prof + 1, (unsigned long long)w_ae);
      atomicAdd(p.prof + 2, (unsigned long long)w_if);
    }
    if (warp == W_MMAB) { atomicAdd(p.prof + 3, (unsigned long long)w_be); atomicAdd(p.prof + 4, (unsigned long long)w_tf); }
    if (warp >= 2 && warp < 2 + 4 * EPG) { atomicAdd(p.prof + 5, (unsigned long long)w_ea); atomicAdd(p.prof + 6, (unsigned long long)w_te); }
    if (warp >= 2 + 4 * EPG && warp < 2 + NEPI) { atomicAdd(p.prof + 7, (unsigned long long)w_eb); atomicAdd(p.prof + 8, (unsigned long long)w_rs); }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace rb
}  // namespace tc

// ---------------------------------------------------------------------------------- host side

static uint16_t rb_bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// sliding-window B image of a C->C conv: per step st (dx-major, K-chunk pair), a block
// [2 K-chunks][3*C rows][8] bf16; row g*C + co = kernel row g, output channel co.
static void rb_pack(const std::vector<float>& w32, const ConvDesc& d, int C, std::vector<uint16_t>& img) {
  const int KC = C / 16, NS = 3 * KC, N = 3 * C;
  const size_t off = img.size();
  img.resize(off + (size_t)NS * N * 16, 0);
  for (int st = 0; st < NS; ++st)
    for (int g = 0; g < 3; ++g)
      for (int co = 0; co < C; ++co)
        for (int k = 0; k < 16; ++k) {
          const int dx = st / KC - 1, ci = 16 * (st % KC) + k;
          const float v = w32[d.w_off + ((size_t)co * d.cin8 * 8 + ci) * 9 + g * 3 + (dx + 1)];
          img[off + (size_t)st * N * 16 + (size_t)(k / 8) * N * 8 + (size_t)(g * C + co) * 8 + (k % 8)] = rb_bf16_bits(v);
        }
}

bool resblock_tc_supported(const SRNet* net, int bin_w) {
  if (net->no_fused_rb) return false;   // REGEN_NO_FUSED_RESBLOCK=1 at create (A/B aid)
  return net->use_tc && bin_w == 128 && (net->cfg.channels == 32 || net->cfg.channels == 16) &&
         net->cfg.n_resblocks > 0 && !net->tc_weights.empty();
}

struct RbImages {
  std::vector<size_t> off;   // byte offset of each resblock's [conv_a | conv_b] image pair
  uint32_t b_bytes = 0;
  uint8_t* d = nullptr;
};

// built once by regen_sr_create (resblock_tc_prepare); launches only read them
static RbImages* rb_images(SRNet* net) {
  if (net->rb_images) return (RbImages*)net->rb_images;
  auto* im = new RbImages();
  const int C = net->cfg.channels;
  std::vector<uint16_t> all;
  for (int b = 0; b < net->cfg.n_resblocks; ++b) {
    const ConvDesc& ca = net->convs[1 + 2 * b];
    const ConvDesc& cb = net->convs[2 + 2 * b];
    im->off.push_back(all.size() * 2);
    rb_pack(net->tc_weights, ca, C, all);
    rb_pack(net->tc_weights, cb, C, all);
  }
  im->b_bytes = (uint32_t)((size_t)3 * (C / 16) * 3 * C * 16 * 2);
  if (cudaMalloc(&im->d, all.size() * 2) != cudaSuccess ||
      cudaMemcpy(im->d, all.data(), all.size() * 2, cudaMemcpyHostToDevice) != cudaSuccess) {
    delete im;
    return nullptr;
  }
  net->rb_images = im;
  return im;
}

regen_status resblock_tc_prepare(SRNet* net) {
  REGEN_REQUIRE(rb_images(net) != nullptr, "fused resblock B images: upload failed");
  return REGEN_OK;
}

void resblock_tc_release(SRNet* net) {
  if (!net->rb_images) return;
  auto* im = (RbImages*)net->rb_images;
  cudaFree(im->d);
  delete im;
  net->rb_images = nullptr;
}

regen_status resblock_tc_launch(const SRNet* cnet, int block, const void* in, void* out, const uint32_t* mbits,
                                int max_bins, const int32_t* d_num_bins, int bin_w, int bin_h, int* counter,
                                cudaStream_t s, int reverse) {
  using namespace tc::rb;
  const SRNet* net = cnet;
  const RbImages* im = (const RbImages*)net->rb_images;
  REGEN_REQUIRE(im != nullptr, "resblock B images not prepared");
  const int C = net->cfg.channels;
  Params p;
  memset(&p, 0, sizeof(p));
  p.in = (const __nv_bfloat16*)in;
  p.out = (__nv_bfloat16*)out;
  p.bias_a = net->d_w32 + net->convs[1 + 2 * block].b_off;
  p.bias_b = net->d_w32 + net->convs[2 + 2 * block].b_off;
  p.mbits = mbits;
  p.num_bins = d_num_bins;
  p.wimg = im->d + im->off[block];
  p.b_bytes = im->b_bytes;
  p.Hr = bin_h;
  p.bin_w = bin_w;
  p.bin_h = bin_h;
  p.max_bins = max_bins;
  p.nbands = (bin_h + BR - 1) / BR;
  p.res_scale = net->cfg.res_scale;
  p.counter = counter;
  p.reverse = reverse;
  {
    const char* dbg = getenv("REGEN_RB_DBG");
    p.dbg = dbg ? atoi(dbg) : 0;
  }
  void (*kern)(Params) = nullptr;
  int G = 0;
  static const int guards = getenv("REGEN_RB_NOGUARD") ? 0 : 1;   // A/B aid: the wrapping ring
  int nslot = 0, nres = 0;
#define RB_PICK(C_, R_, G_, GU_)                                                       \
  {                                                                                   \
    kern = resblock_tc_kernel<C_, R_, G_, GU_>;                                       \
    G = G_;                                                                           \
    nslot = RShape<C_, R_, G_, GU_>::NSLOT;                                           \
    nres = RShape<C_, R_, G_, GU_>::NRES;                                             \
  }
  if (C == 32) {
    if (guards) RB_PICK(32, 6, 1, 2) else RB_PICK(32, 8, 1, 0)
  }
  if (C == 16) {
    if (guards) RB_PICK(16, 12, 1, 2) else RB_PICK(16, 16, 1, 0)
  }
#undef RB_PICK
  REGEN_REQUIRE(kern != nullptr, "fused resblock: unsupported C=%d", C);
  const size_t grp = (size_t)G * (C / 8) * 128 * 16;
  const size_t smem = 1024 + 2ull * nslot * grp + 2ull * p.b_bytes + (size_t)nres * grp;
  REGEN_REQUIRE(smem <= 227 * 1024, "fused resblock SMEM %zu", smem);
  REGEN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::min(max_bins * p.nbands, net->n_sm);
  static unsigned long long* d_prof = nullptr;
  const char* pe = getenv("REGEN_TC_PROF");
  const bool prof = pe && pe[0] == '1';
  if (prof) {
    if (!d_prof) cudaMalloc(&d_prof, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(d_prof, 0, 16 * sizeof(unsigned long long), s);
    p.prof = d_prof;
  }
  REGEN_TRACE("resblock", s);
  kern<<<grid, NTHREADS, smem, s>>>(p);
  REGEN_LAUNCH_CHECK();
  if (prof) {
    unsigned long long h[9];
    cudaMemcpyAsync(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double g = grid;
    fprintf(stderr, "[rb-prof] mma total %.0f | waits a_empty %.0f in_full %.0f b_empty %.0f t_full %.0f | epiA a_full %.0f "
            "t_empty %.0f | epiB b_full %.0f res_full %.0f (cycles/CTA)\n", h[0] / g, h[1] / g, h[2] / g, h[3] / g,
            h[4] / g, h[5] / (4 * EPG * g), h[6] / (4 * EPG * g), h[7] / (4 * EPG * g), h[8] / (4 * EPG * g));
  }
  return REGEN_OK;
}

}  // namespace regen
