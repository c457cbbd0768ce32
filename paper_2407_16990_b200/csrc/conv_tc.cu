// tcgen05 implicit-GEMM 3x3 convolution over packed bins (sm_100a), reading D8/D11 of DESIGN.md.
//
// Layout: activations [bin][row][C/8][Wr][8] bf16 (net.cuh). One bin row of all planes is one
// contiguous run, loaded with a single cp.async.bulk into an SMEM slot with the same layout, which
// IS a K-major no-swizzle UMMA operand: row m (pixel) of a core matrix at +16 B, the two K-chunks
// of an MMA at +LBO (= plane stride), so a dx tap is a +-16 B start-address offset (no im2col).
//
// M = 128 pixels of a row (a "tile"; a row has Wr/128 tiles). Two mappings:
//
//  SLIDE (3*Cout_pad <= 256: head, body, resblock and tail convs). The three kernel rows (dy) are
//   folded into N: one MMA per (dx, K-chunk pair) with N = 3*Cp reads input row r ONCE and adds
//   its contributions to output rows r+1, r, r-1 at the same time. The accumulators of successive
//   output rows sit in TMEM at DEcreasing column addresses (a ring of R slots of Cp columns), so
//   those three rows are one contiguous 3*Cp column window; a window crossing the ring end is split
//   into two MMAs. Slots are pre-filled with the bias by the epilogue (tcgen05.st), so every MMA
//   accumulates. SMEM operand traffic per MMA is 4 KB of A + 3*Cp*32 B of B: at Cp=32 (N=96) the
//   measured SS rate is 56 cyc/MMA vs 48 ideal, vs 46 cyc for N=32 in the plain mapping.
//  PLAIN (the upsampler convs, Cout = C*s^2): output-row accumulator, 9 taps x K-chunk pairs in K,
//   N = a chunk of <= 256 output columns (kept in SMEM per work unit), double-buffered in TMEM.
//
// Warp roles (192 threads, 1 CTA/SM, persistent over work units (bin, band of rows[, N chunk])):
//   warp 0: bulk-copy producer (input rows, B images), warp 1: TMEM alloc + single-thread MMA
//   issuer, warps 2-5: epilogue (TMEM -> regs -> bias/ReLU/residual/mask/pixel-shuffle -> HBM).
//   Pipelines: input-row slots (full/empty mbarriers, released by tcgen05.commit), accumulator
//   slots (full by tcgen05.commit, empty by the 4 epilogue warps), B image (full/empty).
#include <stdlib.h>

#include <vector>

#include "net.cuh"

namespace regen {

namespace tc {

constexpr int NTHREADS = 192;
constexpr int MAX_STEPS = 48;
constexpr int IN_SLOTS = 4;
constexpr int MAX_R = 16;

enum Mode : int { SLIDE = 0, PLAIN = 1 };

struct Step {
  int16_t dx;      // pixel shift of the A start (-1, 0, 1)
  int16_t ky;      // PLAIN: kernel row (input row = y + ky - 1)
  int16_t plane;   // first input plane of the K-chunk pair
  int16_t lbo16;   // 1: LBO = 16 B (chunks are adjacent pixels, head conv); 0: LBO = plane stride
  uint32_t b_off;  // byte offset of this step's B block inside the (chunk's) B image
};

struct Params {
  const __nv_bfloat16* in;
  __nv_bfloat16* out;
  const __nv_bfloat16* skip;
  const float* bias;        // [cout] fp32 (original channel order)
  const int32_t* map;       // [bin][bin_h][bin_w]
  const int32_t* num_bins;
  const uint8_t* wimg;      // B images (global)
  uint32_t b_bytes;         // bytes of one B image (SLIDE: whole conv; PLAIN: one N chunk)
  int mode, role;
  int Wr, Hr, res, bin_w, bin_h;
  int cin8;                 // planes of the input
  int cout;                 // real output channels
  int cp;                   // SLIDE: columns per slot (Cout padded to 16); PLAIN: columns per chunk
  int nchunk;               // PLAIN: N chunks
  int T;                    // tiles per row (Wr / 128)
  int R;                    // SLIDE: TMEM ring slots per tile
  int band;                 // output rows per work unit
  int nbands;
  int max_bins;
  int nsteps;
  int out_c8;               // planes of the output activation (non-HR-output roles)
  int ps;                   // pixel shuffle (UP)
  int C_hr;                 // UP: channels per sub-position (C)
  float res_scale;
  Step steps[MAX_STEPS];
};

// ------------------------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint32_t make_idesc(int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok;
  do {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------------------------- work units
struct Unit {
  int bin, y0, y1, chunk;
};
__device__ __forceinline__ Unit decode_unit(const Params& p, int u) {
  Unit w;
  const int per_chunk = p.max_bins * p.nbands;
  w.chunk = p.mode == PLAIN ? u / per_chunk : 0;
  const int v = u - w.chunk * per_chunk;
  w.bin = v / p.nbands;
  const int band = v - w.bin * p.nbands;
  w.y0 = band * p.band;
  w.y1 = min(p.Hr, w.y0 + p.band);
  return w;
}

// ------------------------------------------------------------------------------- epilogue
// Thread owns pixel x of tile t; v[16] = accumulator columns [c0, c0+16) of output row y.
// SLIDE: columns are output channels (bias already in the accumulator). PLAIN (UP / TINY1): column n
// of chunk j is output column j*cp + n in sub-position-major order (see pack_b_plain).
__device__ __forceinline__ void epilogue_store(const Params& p, const Unit& w, int y, int x, int gcol0, const float* v,
                                               bool occ) {
  const size_t bin_px = (size_t)p.Hr * p.Wr;
  if (p.role == ROLE_TAIL) {
    // HR output [bin][Y][X][4]: channels 0..2 (+ 0 pad); only the first 16-col group holds them
    if (gcol0 != 0) return;
    __nv_bfloat16* o = p.out + ((size_t)w.bin * bin_px + (size_t)y * p.Wr + x) * 4;
    uint2 val;
    val.x = pack_bf16x2(occ ? v[0] : 0.f, occ ? v[1] : 0.f);
    val.y = pack_bf16x2(occ ? v[2] : 0.f, 0.f);
    *reinterpret_cast<uint2*>(o) = val;
    return;
  }
  if (p.role == ROLE_UP || p.role == ROLE_TINY1) {
    // column n -> (sub-position sp = n / Cc, channel c = n % Cc); bias added here (PLAIN)
    const int Cc = p.C_hr;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int n0 = gcol0 + 8 * g;
      const int sp = n0 / Cc, c0 = n0 - sp * Cc;
      if (sp >= p.ps * p.ps) continue;
      const int i = sp / p.ps, jj = sp - i * p.ps;
      const int Y = y * p.ps + i, X = x * p.ps + jj;
      const int Wo = p.Wr * p.ps;
      float r[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int co = (c0 + e) * p.ps * p.ps + sp;   // original (PyTorch) output channel
        const float b = (c0 + e < Cc && co < p.cout) ? __ldg(p.bias + co) : 0.f;
        r[e] = occ ? v[8 * g + e] + b : 0.f;
      }
      if (p.role == ROLE_UP) {
        __nv_bfloat16* o = p.out + (size_t)w.bin * bin_px * p.ps * p.ps * p.out_c8 * 8 +
                           (((size_t)Y * p.out_c8 + c0 / 8) * Wo + X) * 8;
        uint4 val;
        val.x = pack_bf16x2(r[0], r[1]);
        val.y = pack_bf16x2(r[2], r[3]);
        val.z = pack_bf16x2(r[4], r[5]);
        val.w = pack_bf16x2(r[6], r[7]);
        *reinterpret_cast<uint4*>(o) = val;
      } else if (c0 == 0) {
        __nv_bfloat16* o = p.out + ((size_t)w.bin * bin_px * p.ps * p.ps + (size_t)Y * Wo + X) * 4;
        uint2 val;
        val.x = pack_bf16x2(r[0], r[1]);
        val.y = pack_bf16x2(r[2], 0.f);
        *reinterpret_cast<uint2*>(o) = val;
      }
    }
    return;
  }
  // same-resolution activation [bin][y][plane][x][8]
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int c0 = gcol0 + 8 * g;
    if (c0 >= p.cout) continue;
    const size_t idx = (size_t)w.bin * bin_px * p.out_c8 * 8 + (((size_t)y * p.out_c8 + c0 / 8) * p.Wr + x) * 8;
    float r[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) r[e] = v[8 * g + e];
    if (p.role == ROLE_RES_A || p.role == ROLE_TINY0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = fmaxf(r[e], 0.f);
    }
    if (p.role == ROLE_RES_B || p.role == ROLE_BODY) {
      const uint4 sk = *reinterpret_cast<const uint4*>(p.skip + idx);
      const __nv_bfloat162* s2 = reinterpret_cast<const __nv_bfloat162*>(&sk);
      const float sc = p.role == ROLE_RES_B ? p.res_scale : 1.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(s2[e]);
        r[2 * e] = f.x + sc * r[2 * e];
        r[2 * e + 1] = f.y + sc * r[2 * e + 1];
      }
    }
    uint4 val;
    val.x = pack_bf16x2(occ ? r[0] : 0.f, occ ? r[1] : 0.f);
    val.y = pack_bf16x2(occ ? r[2] : 0.f, occ ? r[3] : 0.f);
    val.z = pack_bf16x2(occ ? r[4] : 0.f, occ ? r[5] : 0.f);
    val.w = pack_bf16x2(occ ? r[6] : 0.f, occ ? r[7] : 0.f);
    *reinterpret_cast<uint4*>(p.out + idx) = val;
  }
}

// ------------------------------------------------------------------------------- kernel
__global__ void __launch_bounds__(NTHREADS, 1) conv_tc_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t in_full[IN_SLOTS], in_empty[IN_SLOTS];
  __shared__ __align__(8) uint64_t acc_full[MAX_R], acc_empty[MAX_R];
  __shared__ __align__(8) uint64_t b_full, b_empty;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row_bytes = (uint32_t)p.cin8 * p.Wr * 16;
  // SMEM: [1 KB guard][IN_SLOTS x row_bytes][B image]
  uint8_t* ring = smem_raw + 1024;
  uint8_t* bimg = ring + IN_SLOTS * row_bytes;
  const int nbins = *p.num_bins;
  const int per_chunk = p.max_bins * p.nbands;
  const int total_units = per_chunk * (p.mode == PLAIN ? p.nchunk : 1);
  const int nacc = p.mode == SLIDE ? p.R : 2;   // accumulator slots (per tile)

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < IN_SLOTS; ++i) { mbar_init(&in_full[i], 1); mbar_init(&in_empty[i], 1); }
    for (int i = 0; i < nacc; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
    mbar_init(&b_full, 1);
    mbar_init(&b_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  // SLIDE: pre-fill every accumulator slot with the bias
  if (p.mode == SLIDE && warp >= 2) {
    const int q4 = warp & 3;
    for (int t = 0; t < p.T; ++t)
      for (int s = 0; s < p.R; ++s)
        for (int c0 = 0; c0 < p.cp; c0 += 16) {
          float bv[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) bv[e] = (c0 + e < p.cout) ? __ldg(p.bias + c0 + e) : 0.f;
          tmem_st16(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)((t * p.R + s) * p.cp + c0), bv);
        }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // =============================== producer ===============================
    if (lane == 0) {
      uint32_t rs = 0;          // rows loaded so far (ring sequence)
      int loaded_chunk = -1;
      uint32_t bload = 0;       // B images loaded so far
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const Unit w = decode_unit(p, u);
        if (w.bin >= nbins) continue;
        if (w.chunk != loaded_chunk) {
          if (bload > 0) mbar_wait(&b_empty, (bload - 1) & 1);
          mbar_expect_tx(&b_full, p.b_bytes);
          bulk_g2s(bimg, p.wimg + (size_t)w.chunk * p.b_bytes, p.b_bytes, &b_full);
          ++bload;
          loaded_chunk = w.chunk;
        }
        const int r0 = max(w.y0 - 1, 0), r1 = min(w.y1, p.Hr - 1);
        for (int r = r0; r <= r1; ++r) {
          const uint32_t slot = rs % IN_SLOTS, use = rs / IN_SLOTS;
          mbar_wait(&in_empty[slot], (use & 1) ^ 1);
          mbar_expect_tx(&in_full[slot], row_bytes);
          bulk_g2s(ring + slot * row_bytes, p.in + ((size_t)w.bin * p.Hr + r) * (row_bytes / 2), row_bytes,
                   &in_full[slot]);
          ++rs;
        }
      }
    }
  } else if (warp == 1) {
    // =============================== MMA issuer ===============================
    if (lane == 0) {
      uint32_t rs = 0;     // rows consumed (ring sequence)
      uint32_t q = 0;      // output rows opened (SLIDE: accumulator sequence)
      uint32_t jobs = 0;   // PLAIN: accumulator jobs
      uint32_t bwait = 0;
      int cur_chunk = -1;
      const uint32_t ring_base = smem_u32(ring), b_base = smem_u32(bimg);
      const uint32_t lbo_plane = (uint32_t)p.Wr * 16;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const Unit w = decode_unit(p, u);
        if (w.bin >= nbins) continue;
        if (w.chunk != cur_chunk) {
          if (cur_chunk >= 0) mma_commit(&b_empty);   // previous B image no longer needed
          mbar_wait(&b_full, bwait & 1);
          ++bwait;
          cur_chunk = w.chunk;
          tc_fence_after();
        }
        const int r0 = max(w.y0 - 1, 0), r1 = min(w.y1, p.Hr - 1);
        if (p.mode == SLIDE) {
          const uint32_t Cp = (uint32_t)p.cp;
          const uint32_t q0 = q;   // sequence number of output row y0
          for (int r = r0; r <= r1; ++r) {
            const uint32_t slot = rs % IN_SLOTS;
            mbar_wait(&in_full[slot], (rs / IN_SLOTS) & 1);
            tc_fence_after();
            // window groups g: 0 -> out row r+1, 1 -> r, 2 -> r-1 (kept if inside [y0, y1))
            int g0 = 0, g1 = 3;
            if (r + 1 >= w.y1) g0 = 1;
            if (r >= w.y1) g0 = 2;
            if (r - 1 < w.y0) g1 = 2;
            if (r < w.y0) g1 = 1;
            // open every output row up to the highest one written now (wait until its slot is drained)
            {
              const uint32_t qhi = q0 + (uint32_t)(r + 1 - g0 - w.y0);
              while (q <= qhi) {
                mbar_wait(&acc_empty[q % (uint32_t)p.R], ((q / (uint32_t)p.R) & 1) ^ 1);
                ++q;
              }
            }
            tc_fence_after();
            // column of group g: slot of out row y = r+1-g at (-(q_y)) mod R; groups ascend in columns
            const uint32_t qg0 = q0 + (uint32_t)(r + 1 - g0 - w.y0);   // out row of group g0
            const uint32_t s0 = (uint32_t)((p.R - (int)(qg0 % (uint32_t)p.R)) % p.R);
            const int n_groups = g1 - g0;
            const int first_len = min(n_groups, p.R - (int)s0);   // groups before the ring wraps
            const uint32_t a_row = ring_base + slot * row_bytes;
            for (int t = 0; t < p.T; ++t) {
              const uint32_t tcol = (uint32_t)(t * p.R) * Cp;
              for (int st = 0; st < p.nsteps; ++st) {
                const Step sp = p.steps[st];
                const uint32_t a_addr = a_row + (uint32_t)sp.plane * lbo_plane + (uint32_t)((t * 128 + sp.dx) * 16);
                const uint64_t adesc = make_desc(a_addr, sp.lbo16 ? 16u : lbo_plane, 128);
                const uint32_t bblk = b_base + sp.b_off;
                const uint32_t b_lbo = 3u * Cp * 16u;
                // piece 1: groups [g0, g0 + first_len) at slot s0..
                {
                  const uint64_t bdesc = make_desc(bblk + (uint32_t)g0 * Cp * 16u, b_lbo, 128);
                  mma_bf16(tmem + tcol + s0 * Cp, adesc, bdesc, make_idesc(first_len * (int)Cp), 1u);
                }
                if (first_len < n_groups) {
                  const uint64_t bdesc = make_desc(bblk + (uint32_t)(g0 + first_len) * Cp * 16u, b_lbo, 128);
                  mma_bf16(tmem + tcol, adesc, bdesc, make_idesc((n_groups - first_len) * (int)Cp), 1u);
                }
              }
            }
            mma_commit(&in_empty[slot]);   // input row r fully consumed
            ++rs;
            // output rows completed by this input row: r-1, and r itself at the band/bin end
            if (r - 1 >= w.y0 && r - 1 < w.y1) mma_commit(&acc_full[(q0 + (uint32_t)(r - 1 - w.y0)) % (uint32_t)p.R]);
            if (r == p.Hr - 1 && r >= w.y0 && r < w.y1)
              mma_commit(&acc_full[(q0 + (uint32_t)(r - w.y0)) % (uint32_t)p.R]);
          }
          // rows y1-1 completed by input row y1 (r1 == y1) were committed in the loop
        } else {
          // PLAIN: output row y = sum over ky of input row y+ky-1; rows arrive in order r0..r1
          const uint32_t rs0 = rs;   // ring sequence of row r0
          uint32_t ready = 0;        // rows [r0, r0+ready) known to be in SMEM
          const uint32_t NC = (uint32_t)p.cp;
          for (int y = w.y0; y < w.y1; ++y) {
            const uint32_t ab = jobs & 1, use = jobs >> 1;
            mbar_wait(&acc_empty[ab], (use & 1) ^ 1);
            const int need = min(y + 1, r1);
            while ((int)(r0 + ready) <= need) {
              const uint32_t sq = rs0 + ready;
              mbar_wait(&in_full[sq % IN_SLOTS], (sq / IN_SLOTS) & 1);
              ++ready;
            }
            tc_fence_after();
            for (int t = 0; t < p.T; ++t) {
              uint32_t acc = 0;
              const uint32_t dcol = tmem + ab * (uint32_t)p.T * NC + (uint32_t)t * NC;
              for (int st = 0; st < p.nsteps; ++st) {
                const Step sp = p.steps[st];
                const int r = y + sp.ky - 1;
                if (r < 0 || r >= p.Hr) continue;
                const uint32_t sq = rs0 + (uint32_t)(r - r0);
                const uint32_t a_addr = ring_base + (sq % IN_SLOTS) * row_bytes + (uint32_t)sp.plane * lbo_plane +
                                        (uint32_t)((t * 128 + sp.dx) * 16);
                const uint64_t adesc = make_desc(a_addr, sp.lbo16 ? 16u : lbo_plane, 128);
                const uint64_t bdesc = make_desc(b_base + sp.b_off, NC * 16u, 128);
                mma_bf16(dcol, adesc, bdesc, make_idesc((int)NC), acc);
                acc = 1;
              }
            }
            mma_commit(&acc_full[ab]);
            ++jobs;
            // release input rows whose last reader was this output row
            auto release = [&](int r) {
              if (r < r0 || r > r1) return;
              mma_commit(&in_empty[(rs0 + (uint32_t)(r - r0)) % IN_SLOTS]);
            };
            release(y - 1);
            if (y == w.y1 - 1) { release(y); release(y + 1); }
          }
          rs = rs0 + (uint32_t)(r1 - r0 + 1);
        }
      }
    }
  } else {
    // =============================== epilogue ===============================
    const int q4 = warp & 3;                 // TMEM lane quarter of this warp
    const int m = 32 * q4 + lane;            // pixel within the tile
    const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
    uint32_t q = 0, jobs = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      const Unit w = decode_unit(p, u);
      if (w.bin >= nbins) continue;
      for (int y = w.y0; y < w.y1; ++y) {
        uint32_t s, par, colbase;
        if (p.mode == SLIDE) {
          s = q % (uint32_t)p.R;
          par = (q / (uint32_t)p.R) & 1;
          colbase = (uint32_t)(((p.R - (int)s) % p.R) * p.cp);
        } else {
          s = jobs & 1;
          par = (jobs >> 1) & 1;
          colbase = s * (uint32_t)p.T * (uint32_t)p.cp;
        }
        mbar_wait(&acc_full[s], par);
        tc_fence_after();
        for (int t = 0; t < p.T; ++t) {
          const int x = t * 128 + m;
          const bool occ = p.map[((size_t)w.bin * p.bin_h + y / p.res) * p.bin_w + x / p.res] >= 0;
          const uint32_t tbase = tmem + lane_off +
                                 (p.mode == SLIDE ? (uint32_t)(t * p.R * p.cp) + colbase : colbase + (uint32_t)(t * p.cp));
          const int gbase = p.mode == PLAIN ? w.chunk * p.cp : 0;
          for (int c0 = 0; c0 < p.cp; c0 += 16) {
            float v[16];
            tmem_ld16(tbase + (uint32_t)c0, v);
            epilogue_store(p, w, y, x, gbase + c0, v, occ);
            if (p.mode == SLIDE) {
              float bv[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) bv[e] = (c0 + e < p.cout) ? __ldg(p.bias + c0 + e) : 0.f;
              tmem_st16(tbase + (uint32_t)c0, bv);
            }
          }
        }
        if (p.mode == SLIDE) tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[s]);
        if (p.mode == SLIDE) ++q; else ++jobs;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------- host plans
struct Plan {
  int mode = SLIDE;
  int cp = 0, nchunk = 1, R = 0, nsteps = 0;
  uint32_t b_bytes = 0;
  Step steps[MAX_STEPS];
};

static uint16_t bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// B block of one MMA: [2 K-chunks][N rows][8] bf16 (K-major, no swizzle, SBO 128, LBO N*16)
static void put_b(std::vector<uint16_t>& img, size_t blk_off_elems, int N, int n, int k, float v) {
  img[blk_off_elems + (size_t)(k / 8) * N * 8 + (size_t)n * 8 + (k % 8)] = bf16_bits(v);
}

// W index in the caller's layout [cout][cin][3][3]
static inline float wv(const float* W, int cin, int co, int ci, int ky, int kx) {
  return W[(((size_t)co * cin + ci) * 3 + ky) * 3 + kx];
}

static bool plan_conv(const ConvDesc& d, int C, Plan& pl, std::vector<uint16_t>& img, const float* W) {
  const bool head = d.cin == 3;
  if (!head && d.cin % 16 != 0) return false;
  const int cp16 = (d.cout + 15) / 16 * 16;
  const bool up = d.role == ROLE_UP || d.role == ROLE_TINY1;
  if (!up && 3 * cp16 <= 256) {
    // SLIDE
    pl.mode = SLIDE;
    pl.cp = cp16;
    const int N = 3 * cp16;
    const int T = 1;   // per-tile ring sizing is decided at launch (needs Wr); pick R for the worst T below
    (void)T;
    std::vector<Step> st;
    if (head) {
      // k-step 0: chunks (dx=-1, dx=0); k-step 1: chunks (dx=+1, zeros). LBO = 16 B (adjacent pixels)
      for (int j = 0; j < 2; ++j) {
        Step s{};
        s.dx = j == 0 ? -1 : 1;
        s.ky = 0;
        s.plane = 0;
        s.lbo16 = 1;
        s.b_off = (uint32_t)(j * N * 32);
        st.push_back(s);
      }
    } else {
      for (int dx = -1; dx <= 1; ++dx)
        for (int kc = 0; kc < d.cin / 16; ++kc) {
          Step s{};
          s.dx = (int16_t)dx;
          s.ky = 0;
          s.plane = (int16_t)(2 * kc);
          s.lbo16 = 0;
          s.b_off = (uint32_t)(st.size() * N * 32);
          st.push_back(s);
        }
    }
    pl.nsteps = (int)st.size();
    for (int i = 0; i < pl.nsteps; ++i) pl.steps[i] = st[i];
    img.assign((size_t)pl.nsteps * N * 16, 0);
    for (int i = 0; i < pl.nsteps; ++i) {
      const size_t base = (size_t)i * N * 16;
      for (int g = 0; g < 3; ++g)            // group g = kernel row ky = g (out row r+1-g <- dy = g-1)
        for (int co = 0; co < d.cout; ++co)
          for (int k = 0; k < 16; ++k) {
            float v = 0.f;
            if (head) {
              const int dx = i == 0 ? (k < 8 ? -1 : 0) : (k < 8 ? 1 : 99);
              const int ci = k % 8;
              if (dx != 99 && ci < 3) v = wv(W, 3, co, ci, g, dx + 1);
            } else {
              const int ci = 16 * (st[i].plane / 2) + k;
              v = wv(W, d.cin, co, ci, g, st[i].dx + 1);
            }
            put_b(img, base, N, g * cp16 + co, k, v);
          }
    }
    pl.b_bytes = (uint32_t)(img.size() * 2);
    return true;
  }
  if (!up || head) return false;
  // PLAIN (upsampler): TMEM column n = sp * C + c  <-> original channel co = c * s^2 + sp
  const int s2 = d.ps * d.ps;
  const int Cc = d.cout / s2;
  int NC = 0;
  for (int cand : {256, 192, 144, 128, 96, 64, 48, 32, 16}) {
    if (d.cout % cand == 0 && (size_t)9 * (d.cin / 16) * cand * 32 <= 150 * 1024) { NC = cand; break; }
  }
  if (d.role != ROLE_UP || NC == 0) return false;   // TINY1 (3 channels per sub-position) stays on SIMT
  pl.mode = PLAIN;
  pl.cp = NC;
  pl.nchunk = (d.cout + NC - 1) / NC;
  std::vector<Step> st;
  for (int ky = 0; ky < 3; ++ky)
    for (int dx = -1; dx <= 1; ++dx)
      for (int kc = 0; kc < d.cin / 16; ++kc) {
        Step s{};
        s.dx = (int16_t)dx;
        s.ky = (int16_t)ky;
        s.plane = (int16_t)(2 * kc);
        s.lbo16 = 0;
        s.b_off = (uint32_t)(st.size() * NC * 32);
        st.push_back(s);
      }
  if ((int)st.size() > MAX_STEPS) return false;
  pl.nsteps = (int)st.size();
  for (int i = 0; i < pl.nsteps; ++i) pl.steps[i] = st[i];
  const size_t chunk_elems = (size_t)pl.nsteps * NC * 16;
  img.assign(chunk_elems * pl.nchunk, 0);
  for (int j = 0; j < pl.nchunk; ++j)
    for (int i = 0; i < pl.nsteps; ++i) {
      const size_t base = j * chunk_elems + (size_t)i * NC * 16;
      for (int n = 0; n < NC; ++n) {
        const int col = j * NC + n;
        const int sp = col / Cc, c = col % Cc;
        if (sp >= s2) continue;
        const int co = c * s2 + sp;
        for (int k = 0; k < 16; ++k) {
          const int ci = 16 * (st[i].plane / 2) + k;
          put_b(img, base, NC, n, k, wv(W, d.cin, co, ci, st[i].ky, st[i].dx + 1));
        }
      }
    }
  pl.b_bytes = (uint32_t)(chunk_elems * 2);
  return true;
}

struct NetPlans {
  std::vector<Plan> plans;   // per conv (mode/cp/...); plans[i].nsteps == 0 => SIMT
};

}  // namespace tc

float round_bf16_host(float f);

// Weights in the caller order are needed to build the B images: rebuild them from d_w32.
regen_status conv_tc_prepare(SRNet* net) {
  using namespace tc;
  net->use_tc = false;
  if (net->cfg.dtype != REGEN_DTYPE_BF16 || net->cfg.channels % 16 != 0) return REGEN_OK;
  const char* force = getenv("REGEN_FORCE_SIMT");   // debugging aid: run every conv on the SIMT kernel
  if (force && force[0] == '1') return REGEN_OK;
  // fetch the (bf16-rounded, zero-padded) fp32 weights back and repack
  size_t total = 0;
  for (auto& d : net->convs) total = std::max(total, d.b_off + (size_t)d.cout);
  std::vector<float> w32(total);
  cudaError_t e = cudaMemcpy(w32.data(), net->d_w32, total * sizeof(float), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    set_error("weights readback: %s", cudaGetErrorString(e));
    return REGEN_E_CUDA;
  }
  std::vector<uint8_t> all;
  auto* plans = new NetPlans();
  for (auto& d : net->convs) {
    // caller-order view [cout][cin][3][3] from the padded [cout][cin8*8][9]
    std::vector<float> W((size_t)d.cout * d.cin * 9);
    for (int co = 0; co < d.cout; ++co)
      for (int ci = 0; ci < d.cin; ++ci)
        for (int t = 0; t < 9; ++t) W[((size_t)co * d.cin + ci) * 9 + t] = w32[d.w_off + ((size_t)co * d.cin8 * 8 + ci) * 9 + t];
    Plan pl;
    std::vector<uint16_t> img;
    if (plan_conv(d, net->cfg.channels, pl, img, W.data())) {
      d.tc_mode = pl.mode + 1;
      all.resize((all.size() + 1023) / 1024 * 1024);
      d.tc_off = all.size();
      const uint8_t* b = reinterpret_cast<const uint8_t*>(img.data());
      all.insert(all.end(), b, b + img.size() * 2);
    } else {
      d.tc_mode = 0;
      pl.nsteps = 0;
    }
    plans->plans.push_back(pl);
  }
  if (!all.empty()) {
    e = cudaMalloc(&net->d_wtc, all.size());
    if (e == cudaSuccess) e = cudaMemcpy(net->d_wtc, all.data(), all.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      set_error("B image upload: %s", cudaGetErrorString(e));
      delete plans;
      return REGEN_E_CUDA;
    }
    net->wtc_bytes = all.size();
  }
  net->tc_plans = plans;
  net->use_tc = true;
  return REGEN_OK;
}

void conv_tc_release(SRNet* net) {
  delete (tc::NetPlans*)net->tc_plans;
  net->tc_plans = nullptr;
}

bool conv_tc_supported(const SRNet* net, const ConvDesc& cv) { return net->use_tc && cv.tc_mode != 0; }

regen_status conv_tc_launch(const SRNet* net, const ConvDesc& cv, const void* in, void* out, const void* skip,
                            const int32_t* map, int max_bins, const int32_t* d_num_bins, int bin_w, int bin_h,
                            cudaStream_t s) {
  using namespace tc;
  const NetPlans* np = (const NetPlans*)net->tc_plans;
  const size_t idx = &cv - net->convs.data();
  const Plan& pl = np->plans[idx];
  Params p;
  memset(&p, 0, sizeof(p));
  p.in = (const __nv_bfloat16*)in;
  p.out = (__nv_bfloat16*)out;
  p.skip = (const __nv_bfloat16*)skip;
  p.bias = net->d_w32 + cv.b_off;
  p.map = map;
  p.num_bins = d_num_bins;
  p.wimg = net->d_wtc + cv.tc_off;
  p.b_bytes = pl.b_bytes;
  p.mode = pl.mode;
  p.role = cv.role;
  p.Wr = bin_w * cv.res;
  p.Hr = bin_h * cv.res;
  p.res = cv.res;
  p.bin_w = bin_w;
  p.bin_h = bin_h;
  p.cin8 = cv.cin8;
  p.cout = cv.cout;
  p.cp = pl.cp;
  p.nchunk = pl.nchunk;
  REGEN_REQUIRE(p.Wr % 128 == 0, "tcgen05 conv needs bin width*res multiple of 128 (got %d)", p.Wr);
  p.T = p.Wr / 128;
  if (pl.mode == SLIDE) {
    int R = MAX_R;
    while (R > 4 && p.T * R * p.cp > 512) R >>= 1;
    REGEN_REQUIRE(p.T * R * p.cp <= 512 && R >= 4, "TMEM ring does not fit (T=%d cp=%d)", p.T, p.cp);
    p.R = R;
  } else {
    REGEN_REQUIRE(2 * p.T * p.cp <= 512, "TMEM double buffer does not fit (T=%d NC=%d)", p.T, p.cp);
    p.R = 2;
  }
  p.band = 32;
  p.nbands = (p.Hr + p.band - 1) / p.band;
  p.max_bins = max_bins;
  p.nsteps = pl.nsteps;
  memcpy(p.steps, pl.steps, sizeof(Step) * pl.nsteps);
  p.ps = cv.ps;
  p.C_hr = (cv.role == ROLE_UP || cv.role == ROLE_TINY1) ? cv.cout / (cv.ps * cv.ps) : 0;
  p.out_c8 = cv.role == ROLE_UP ? (p.C_hr + 7) / 8 : (cv.cout + 7) / 8;
  p.res_scale = cv.role == ROLE_RES_B ? net->cfg.res_scale : 1.0f;
  const uint32_t row_bytes = (uint32_t)p.cin8 * p.Wr * 16;
  const size_t smem = 1024 + (size_t)IN_SLOTS * row_bytes + pl.b_bytes;
  REGEN_REQUIRE(smem <= 227 * 1024, "conv SMEM %zu too large", smem);
  REGEN_CUDA(cudaFuncSetAttribute(conv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  static int nsm = 0;
  if (nsm == 0) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int units = max_bins * p.nbands * (pl.mode == PLAIN ? pl.nchunk : 1);
  const int grid = std::min(units, nsm);
  conv_tc_kernel<<<grid, NTHREADS, smem, s>>>(p);
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

}  // namespace regen
