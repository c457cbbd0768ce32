// a8: scatter-and-blend, eq. P:461-464 "SR(MB_s) + IN(unselected MBs)", "stitching them
// back to bi-linear-interpolated non-regions". Every HR pixel is written exactly once: the bilinear
// value (D10: half-pixel centres, edge clamp, fp32) or, inside the HR square of an owned selected MB,
// the box's HR bin pixel (un-rotated, D7). Stores are 16-B vectors; u8 frames (D20) quantise in integers.
#include <algorithm>
#include <stdlib.h>
#include <string.h>

#include "net.cuh"

namespace regen {

template <typename T>
__device__ __forceinline__ float ld_hr(const T* p);
template <>
__device__ __forceinline__ float ld_hr<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_hr<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

enum { SC_ALL = 0, SC_BILINEAR = 1, SC_OWNED = 2 };

struct ScatterArgs {
  const uint8_t* frames;
  const regen_box* boxes;
  const int32_t* owner;
  const void* hr;
  void* out;
  int W, H, OW, OH, GW, GH, mb, s, bin_w, bin_h;
  float inv_s;
  int mode;         // SC_ALL, SC_BILINEAR (owned MBs written elsewhere: the fold combine), SC_OWNED
  int64_t n_frames;
  int format;       // REGEN_FORMAT_RGB8 / NV12 (converted while the LR pixels are read, D19)
};

// One CTA per (frame, LR row y) writes the S HR rows S*y .. S*y+S-1. The (at most three) LR rows
// they interpolate from (16-B loads) and the owner row of their MB row go to SMEM once; then per HR
// row: (1) vertical pass -> SMEM [W] float4; (2) horizontal pass, a thread per pair of LR columns
// computing their 2*S HR pixels (6*S values = whole 32-bit words, consecutive threads ->
// consecutive words: no bank conflicts) into an SMEM copy of the output row, with the D10 weights
// of each sub-pixel phase compile-time (HR pixel X = S*x + j samples src = x + (j + 0.5)/S - 0.5:
// columns (x-1, x) or (x, x+1) with a fixed fraction, clamped at the edges exactly as the oracle);
// (3) coalesced 16-B copy-out (an MB's HR square is a whole number of chunks) skipping owned MB
// squares, which get the owner box's HR bin pixels (SC_ALL, SC_OWNED) or nothing (SC_BILINEAR:
// regen_enhance_scatter wrote them already). ~28 KB SMEM per CTA: 8 CTAs per SM.
// 128 threads x <= 64 registers and ~28 KB SMEM per CTA, so a CTA fits beside a resident SR conv
// CTA (the bilinear pass of batch k+1 runs concurrently with the SR of batch k, schedule.py)
constexpr int SC_THREADS = 128;

template <int S>
struct Phase {   // sub-pixel phase j: source offset d (-1 or 0) and fraction
  __host__ __device__ static constexpr int d(int j) { return 2 * j + 1 < S ? -1 : 0; }
  __host__ __device__ static constexpr float f(int j) {
    return 2 * j + 1 < S ? (float)(1.0 + ((j + 0.5) / S - 0.5)) : (float)((j + 0.5) / S - 0.5);
  }
  // the fraction as an exact numerator over 2S (D20's integer form): f(j) = num(j) / (2S)
  __host__ __device__ static constexpr int num(int j) { return 2 * j + 1 < S ? 2 * j + 1 + S : 2 * j + 1 - S; }
};

template <typename TO>
__device__ __forceinline__ void put2(uint32_t* w, int k, float a, float b);
template <>
__device__ __forceinline__ void put2<__nv_bfloat16>(uint32_t* w, int k, float a, float b) { w[k] = pack_bf16(a, b); }
template <>
__device__ __forceinline__ void put2<float>(uint32_t* w, int k, float a, float b) {
  w[2 * k] = __float_as_uint(a);
  w[2 * k + 1] = __float_as_uint(b);
}

template <int S, typename TH, typename TO, int MODE>
__global__ void __launch_bounds__(SC_THREADS, 8) scatter_rows_kernel(ScatterArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int64_t sf = blockIdx.y;
  const int y = blockIdx.x;
  const int W = a.W, W3 = W * 3;
  constexpr bool U8 = sizeof(TO) == 1;
  constexpr int CPT = U8 ? 4 : 2;                                             // LR columns per thread
  const int npair = (W + CPT - 1) / CPT;
  constexpr int WPP = 3 * S * CPT * (int)sizeof(TO) / 4;                      // 32-bit words per unit
  const int row_words = (npair * WPP + 3) / 4 * 4;                            // staging row (16-B multiple)
  const int W3p = (W3 + 15) / 16 * 16;
  float4* vr = reinterpret_cast<float4*>(sm);                                 // [W]
  uint32_t* orow = reinterpret_cast<uint32_t*>(vr + W);                       // [row_words]
  int32_t* own = reinterpret_cast<int32_t*>(orow + row_words);                // [GW (+pad)]
  uint8_t* lr = reinterpret_cast<uint8_t*>(own + (a.GW + 3) / 4 * 4);         // [3][W3p]
  const uint8_t* img = a.frames + sf * (int64_t)a.H * W3;
  // ---- 0. the (at most three) LR rows (16-B loads when aligned) and the owner row -> SMEM
  for (int k = 0; k < (MODE == SC_OWNED ? 0 : 3); ++k) {
    const uint8_t* src = img + (size_t)min(max(y - 1 + k, 0), a.H - 1) * W3;
    uint8_t* dst = lr + k * W3p;
    if (a.format == REGEN_FORMAT_NV12) {   // NV12 -> RGB8 row in SMEM
      for (int j = threadIdx.x; j < W; j += SC_THREADS) {
        int cr, cg, cb;
        frame_px(a.frames, REGEN_FORMAT_NV12, sf, W, a.H, j, min(max(y - 1 + k, 0), a.H - 1), cr, cg, cb);
        dst[3 * j] = (uint8_t)cr;
        dst[3 * j + 1] = (uint8_t)cg;
        dst[3 * j + 2] = (uint8_t)cb;
      }
      continue;
    }
    if ((((uintptr_t)src) & 15) == 0) {
      for (int j = threadIdx.x; j < W3 / 16; j += SC_THREADS)
        reinterpret_cast<uint4*>(dst)[j] = __ldg(reinterpret_cast<const uint4*>(src) + j);
      for (int j = W3 / 16 * 16 + threadIdx.x; j < W3; j += SC_THREADS) dst[j] = src[j];
    } else {
      for (int j = threadIdx.x; j < W3; j += SC_THREADS) dst[j] = src[j];
    }
  }
  const int my = y / a.mb;   // MB row of all S HR rows
  for (int j = threadIdx.x; j < a.GW; j += SC_THREADS) own[j] = a.owner[(sf * a.GH + my) * a.GW + j];
  constexpr int MB_BYTES = 16 * S * 3 * (int)sizeof(TO);     // HR width of an MB in bytes (mb = 16)
  static_assert(MB_BYTES % 16 == 0, "MB squares must be whole 16-B chunks");
  const int row_bytes = a.OW * 3 * (int)sizeof(TO);
  const int n16 = row_bytes / 16;
  if (MODE == SC_OWNED) __syncthreads();   // owner row staged
#pragma unroll
  for (int i = 0; i < (MODE == SC_OWNED ? 0 : S); ++i) {
    const int Y = y * S + i;
    // ---- 1. vertical pass (D10) of HR row i
    int yl0 = y + Phase<S>::d(i);
    float ly = Phase<S>::f(i);
    if (yl0 < 0) { yl0 = 0; ly = 0.f; }
    const int yl1 = min(yl0 + 1, a.H - 1);
    if (yl1 == yl0) ly = 0.f;
    __syncthreads();   // LR rows staged / previous row's horizontal pass done
    {
      const uint8_t* r0 = lr + (yl0 - (y - 1)) * W3p;   // slot k holds row clamp(y-1+k)
      const uint8_t* r1 = lr + (yl1 - (y - 1)) * W3p;
      if constexpr (U8) {   // D20: exact integer vertical sums 2S p0 + b (p1 - p0), ly = b / (2S), in fp32
        const float b = ly == 0.f ? 0.f : (float)Phase<S>::num(i);   // ly == 0: the edge clamps (above)
        for (int x = threadIdx.x; x < W; x += SC_THREADS) {
          float4 v;
          float p0 = (float)r0[3 * x], p1 = (float)r1[3 * x];
          v.x = fmaf(b, p1 - p0, (float)(2 * S) * p0);
          p0 = (float)r0[3 * x + 1]; p1 = (float)r1[3 * x + 1];
          v.y = fmaf(b, p1 - p0, (float)(2 * S) * p0);
          p0 = (float)r0[3 * x + 2]; p1 = (float)r1[3 * x + 2];
          v.z = fmaf(b, p1 - p0, (float)(2 * S) * p0);
          v.w = 0.f;
          vr[x] = v;
        }
      } else
      for (int x = threadIdx.x; x < W; x += SC_THREADS) {
        float4 v;   // pre-scaled by 1/255 (the same arithmetic as bilinear_kernel: bit-identical pixels)
        float p0 = (float)r0[3 * x], p1 = (float)r1[3 * x];
        v.x = __fmul_rn(fmaf(ly, p1 - p0, p0), 1.0f / 255.0f);
        p0 = (float)r0[3 * x + 1]; p1 = (float)r1[3 * x + 1];
        v.y = __fmul_rn(fmaf(ly, p1 - p0, p0), 1.0f / 255.0f);
        p0 = (float)r0[3 * x + 2]; p1 = (float)r1[3 * x + 2];
        v.z = __fmul_rn(fmaf(ly, p1 - p0, p0), 1.0f / 255.0f);
        v.w = 0.f;
        vr[x] = v;
      }
    }
    __syncthreads();   // vr ready; previous row's copy-out done
    // ---- 2. horizontal pass: a thread per pair of LR columns -> 2*S HR pixels (6*S values, whole
    // 32-bit words; consecutive threads -> consecutive words: no bank conflicts)
    if constexpr (U8) {   // D20: a thread per 4 LR columns -> 4*S HR pixels = 3*S words
      constexpr float invD = 1.0f / (float)(4 * S * S);
      for (int t = threadIdx.x; t < npair; t += SC_THREADS) {
        const int x0 = 4 * t;
        float4 v[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) v[q] = vr[min(max(x0 - 1 + q, 0), W - 1)];
        uint32_t o[12 * S];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int x = x0 + q;
#pragma unroll
          for (int j = 0; j < S; ++j) {
            float4 A, B;
            float n = (float)Phase<S>::num(j);
            if (Phase<S>::d(j) < 0) {
              A = v[q]; B = v[q + 1];
              if (x == 0) { n = 0.f; A = v[q + 1]; }
            } else {
              A = v[q + 1]; B = v[q + 2];
              if (x >= W - 1) n = 0.f;
            }
            const int e = 3 * (q * S + j);   // n = 2S A + num (B - A): exact integers in fp32
            o[e] = u8_code(fmaf(n, B.x - A.x, (float)(2 * S) * A.x), invD);
            o[e + 1] = u8_code(fmaf(n, B.y - A.y, (float)(2 * S) * A.y), invD);
            o[e + 2] = u8_code(fmaf(n, B.z - A.z, (float)(2 * S) * A.z), invD);
          }
        }
#pragma unroll
        for (int k = 0; k < WPP; ++k) orow[t * WPP + k] = pack_u8x4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
      }
    } else
    for (int t = threadIdx.x; t < npair; t += SC_THREADS) {
      const int x0 = 2 * t;
      float4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = vr[min(max(x0 - 1 + q, 0), W - 1)];
      float o[6 * S];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int x = x0 + q;
#pragma unroll
        for (int j = 0; j < S; ++j) {
          float4 A, B;
          float lx = Phase<S>::f(j);
          if (Phase<S>::d(j) < 0) {
            A = v[q]; B = v[q + 1];
            if (x == 0) { lx = 0.f; A = v[q + 1]; }   // src < 0 clamps to column 0
          } else {
            A = v[q + 1]; B = v[q + 2];
            if (x >= W - 1) lx = 0.f;                 // last column: i1 = i0
          }
          const int e = 3 * (q * S + j);
          // explicit rounding (no FMA contraction across the steps): bit-identical to bilinear_kernel
          o[e] = fmaf(lx, __fsub_rn(B.x, A.x), A.x);
          o[e + 1] = fmaf(lx, __fsub_rn(B.y, A.y), A.y);
          o[e + 2] = fmaf(lx, __fsub_rn(B.z, A.z), A.z);
        }
      }
      uint32_t w[WPP];
#pragma unroll
      for (int k = 0; k < 3 * S; ++k) put2<TO>(w, k, o[2 * k], o[2 * k + 1]);
#pragma unroll
      for (int k = 0; k < WPP; ++k) orow[t * WPP + k] = w[k];
    }
    __syncthreads();
    // ---- 3. copy-out of HR row i in coalesced 16-B chunks, owned MB squares skipped
    uint8_t* drow = (uint8_t*)a.out + ((sf * a.OH + Y) * (int64_t)a.OW) * 3 * sizeof(TO);
    const uint8_t* srow = reinterpret_cast<const uint8_t*>(orow);
    if ((((uintptr_t)drow) & 15) == 0) {
      for (int c = threadIdx.x; c < n16; c += SC_THREADS) {
        if (own[(c * 16) / MB_BYTES] >= 0) continue;
        *reinterpret_cast<uint4*>(drow + 16 * c) = *reinterpret_cast<const uint4*>(srow + 16 * c);
      }
      for (int c = n16 * 16 + threadIdx.x; c < row_bytes; c += SC_THREADS)
        if (own[c / MB_BYTES] < 0) drow[c] = srow[c];
    } else if (U8) {
      for (int c = threadIdx.x; c < row_bytes; c += SC_THREADS)
        if (own[c / MB_BYTES] < 0) drow[c] = srow[c];
    } else {
      for (int c = threadIdx.x; c < row_bytes / 2; c += SC_THREADS)
        if (own[(2 * c) / MB_BYTES] < 0) reinterpret_cast<uint16_t*>(drow)[c] = reinterpret_cast<const uint16_t*>(srow)[c];
    }
  }
  if (MODE == SC_BILINEAR) return;
  // ---- owned MBs: the box's HR bin pixels (un-rotated, D7), 8 pixels per thread
  const int HW = S * a.bin_w, HH = S * a.bin_h;
  const int nchunk = (a.OW + 7) / 8;
  for (int t = threadIdx.x; t < S * nchunk; t += SC_THREADS) {
    const int i = t / nchunk, c = t - i * nchunk;
    const int Y = y * S + i;
    const int X0 = c * 8;
    const int32_t b = own[X0 / (16 * S)];   // the 8 pixels lie in one MB column (16*S is a multiple of 8)
    if (b < 0) continue;
    const regen_box* bp = a.boxes + b;
    const int x0 = bp->x0, y0 = bp->y0, hh = bp->h, bin = bp->bin, bbx = bp->bx, bby = bp->by, rot = bp->rotated;
    const int u0 = X0 - S * x0, v = Y - S * y0;
    const TH* hb = (const TH*)a.hr + (size_t)bin * HH * HW * 4;
    // rotated 90 deg CW: box-local (u, v) <- bin (S*h-1-v, u)
    const TH* src = !rot ? hb + ((size_t)(S * bby + v) * HW + S * bbx + u0) * 4
                         : hb + ((size_t)(S * bby + u0) * HW + S * bbx + (S * hh - 1 - v)) * 4;
    const size_t step = !rot ? 4 : (size_t)HW * 4;
    TO* dst = (TO*)a.out + ((sf * a.OH + Y) * (int64_t)a.OW + X0) * 3;
    for (int k = 0; k < 8 && X0 + k < a.OW; ++k) {
      float f0, f1, f2;
      if (sizeof(TH) == 2) {
        const uint2 q = *reinterpret_cast<const uint2*>(src + (size_t)k * step);
        const float2 f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.x));
        const float2 f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.y));
        f0 = f01.x; f1 = f01.y; f2 = f23.x;
      } else {
        const float4 f = *reinterpret_cast<const float4*>(src + (size_t)k * step);
        f0 = f.x; f1 = f.y; f2 = f.z;
      }
      if (U8) {   // D20: the model-dtype value, quantised
        ((uint8_t*)dst)[3 * k] = (uint8_t)q_u8(f0);
        ((uint8_t*)dst)[3 * k + 1] = (uint8_t)q_u8(f1);
        ((uint8_t*)dst)[3 * k + 2] = (uint8_t)q_u8(f2);
      } else if (sizeof(TO) == 2) {
        ((__nv_bfloat16*)dst)[3 * k] = __float2bfloat16_rn(f0);
        ((__nv_bfloat16*)dst)[3 * k + 1] = __float2bfloat16_rn(f1);
        ((__nv_bfloat16*)dst)[3 * k + 2] = __float2bfloat16_rn(f2);
      } else {
        ((float*)dst)[3 * k] = f0;
        ((float*)dst)[3 * k + 1] = f1;
        ((float*)dst)[3 * k + 2] = f2;
      }
    }
  }
}


// ---------------------------------------------------------------------------------------------
// Bilinear-only pass (SC_BILINEAR; frame width a multiple of 8): a warp per (frame, HR row, 32 groups
// of 8 LR columns); a lane computes the 8*S HR pixels of its group in registers — LR bytes read as
// aligned 32-bit words (the group's 10 columns x 3 channels sit at a fixed byte offset 1 inside 9
// words: 3*x0 - 4 is word aligned because x0 is a multiple of 8), vertical then horizontal D10 lerp
// at compile-time phases — and stages them in SMEM; the warp then writes its contiguous run of the HR
// row with coalesced 16-B stores (lane k -> chunk k), skipping groups in owned MBs (an MB is 16 LR
// columns: a group never straddles one). The first and last group of a row take a clamped path.
constexpr int BL_WARPS = 4;

// packed fp32x2 arithmetic (sm_100: FADD2 / FFMA2 / FMUL2), round-to-nearest per element
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ float f2lo(unsigned long long v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ unsigned long long f2sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// The 8 words holding LR columns x0-1 .. x0+8 of a row at bytes 1 + 3c (c = 0..9), x0 a multiple of 8;
// the edge clamps (column -1 -> 0 at x0 = 0, column W -> W-1 at x0 = W-8) are built by word moves, so
// the first and last group of a row take the same instructions as the others (no divergent clamped path
// in their warps). `row` = the LR row's first byte, 4-B aligned; W >= 16.
__device__ __forceinline__ void row_window(const uint8_t* row, int x0, int W, uint32_t (&u)[8]) {
  const bool left = x0 == 0, right = x0 + 9 > W;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(left ? row : row + 3 * x0 - 4);
  uint32_t t[8];
#pragma unroll
  for (int k = 0; k < 7; ++k) t[k] = __ldg(w + k);
  t[7] = right ? 0u : __ldg(w + 7);   // past the row at the right edge: not loaded
  u[0] = left ? t[0] << 8 : t[0];     // window byte b = row byte b - 4 at the left edge, col -1 = col 0
#pragma unroll
  for (int k = 1; k < 7; ++k) u[k] = left ? t[k - 1] : t[k];
  u[7] = left ? t[6] : (right ? t[6] >> 8 : t[7]);   // right edge: col x0+8 = col x0+7 (bytes 25..27)
}

template <int S, typename TO>
struct BL {
  static constexpr int VALS = 8 * S * 3;                        // values per group
  static constexpr int BYTES = VALS * (int)sizeof(TO);          // 144 B at S = 3, bf16
  static constexpr int CHUNKS = BYTES / 16;
  static_assert(BYTES % 16 == 0, "group bytes");
};

template <int S, typename TO>
__global__ void __launch_bounds__(32 * BL_WARPS, 8) bilinear_kernel(ScatterArgs a, int nwc) {
  extern __shared__ __align__(16) uint8_t bsm[];
  using G = BL<S, TO>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* stage = bsm + warp * 32 * G::BYTES;
  const int W = a.W, W3 = 3 * W, GW = a.GW;
  const int ngroups = W / 8;
  // 32-bit item arithmetic (the host launches this kernel only for < 2^31 items): two 32-bit divisions
  // per item instead of two calls of the 64-bit division routine
  const uint32_t n_items = (uint32_t)((int64_t)a.n_frames * a.OH * nwc);
  for (uint32_t it = blockIdx.x * BL_WARPS + warp; it < n_items; it += gridDim.x * BL_WARPS) {
    const uint32_t rowi32 = it / (uint32_t)nwc;
    const int wc = (int)(it - rowi32 * (uint32_t)nwc);
    const uint32_t f32 = rowi32 / (uint32_t)a.OH;
    const int64_t rowi = rowi32;             // frame * OH + Y
    const int Y = (int)(rowi32 - f32 * (uint32_t)a.OH);
    const int64_t f = f32;
    const int g = wc * 32 + lane;
    const int x0 = 8 * g;
    const int my = (Y / S) / 16;
    bool act = g < ngroups;
    if (act) act = __ldg(a.owner + (f * a.GH + my) * GW + x0 / 16) < 0;
    const uint32_t amask = __ballot_sync(0xffffffffu, act);
    if (amask == 0u) continue;
    if (act) {
      // vertical pass: HR row Y = S*y + i samples LR rows (yl0, yl1) at fraction ly (D10)
      const int y = Y / S, i = Y - y * S;
      int yl0 = y + (2 * i + 1 < S ? -1 : 0);
      float ly = 0.f;
#pragma unroll
      for (int q = 0; q < S; ++q)
        if (q == i) ly = Phase<S>::f(q);
      if (yl0 < 0) { yl0 = 0; ly = 0.f; }
      const int yl1 = min(yl0 + 1, a.H - 1);
      if (yl1 == yl0) ly = 0.f;
      const uint8_t* r0 = a.frames + (f * a.H + yl0) * (int64_t)W3;
      const uint8_t* r1 = a.frames + (f * a.H + yl1) * (int64_t)W3;
      // LR columns x0-1 .. x0+8 after the vertical lerp, pre-scaled by 1/255, and the differences
      // of neighbouring columns: each HR value is then one FMA (or a copy at fraction 0)
      float vr[10][3];
      if (a.format == REGEN_FORMAT_RGB8 && W >= 16 && ((((uintptr_t)r0) | ((uintptr_t)r1)) & 3) == 0) {
        uint32_t u0[8], u1[8];
        if (ly == 0.f) {   // the HR row sits on LR row yl0 (phase fraction 0, or an edge clamp): one row
          row_window(r0, x0, W, u0);
#pragma unroll
          for (int c = 0; c < 10; ++c)
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              const int b = 1 + 3 * c + ch;
              const float p0 = __uint_as_float(__byte_perm(u0[b >> 2], 0x4B000000u, 0x7650u | (b & 3))) - 8388608.0f;
              vr[c][ch] = __fmul_rn(p0, 1.0f / 255.0f);   // == fmaf(0, p1 - p0, p0) / 255 exactly
            }
        } else {
          row_window(r0, x0, W, u0);
          row_window(r1, x0, W, u1);
          // the 30 values as 15 pairs, each step one packed fp32x2 instruction (FADD2/FFMA2/FMUL2:
          // per-element IEEE round-to-nearest, bit-identical to the scalar chain of the row kernel)
          float* vf = &vr[0][0];
          const unsigned long long m23 = f2pack(8388608.0f, 8388608.0f), k255 = f2pack(1.0f / 255.0f, 1.0f / 255.0f);
          const unsigned long long ly2 = f2pack(ly, ly);
#pragma unroll
          for (int e = 0; e < 30; e += 2) {
            const int b0 = 1 + e, b1 = 2 + e;   // bytes within the words (compile-time)
            const unsigned long long q0 = f2pack(__uint_as_float(__byte_perm(u0[b0 >> 2], 0x4B000000u, 0x7650u | (b0 & 3))),
                                                 __uint_as_float(__byte_perm(u0[b1 >> 2], 0x4B000000u, 0x7650u | (b1 & 3))));
            const unsigned long long q1 = f2pack(__uint_as_float(__byte_perm(u1[b0 >> 2], 0x4B000000u, 0x7650u | (b0 & 3))),
                                                 __uint_as_float(__byte_perm(u1[b1 >> 2], 0x4B000000u, 0x7650u | (b1 & 3))));
            const unsigned long long p0 = f2sub(q0, m23), p1 = f2sub(q1, m23);
            const unsigned long long r = f2mul(f2fma(ly2, f2sub(p1, p0), p0), k255);
            vf[e] = f2lo(r);
            vf[e + 1] = f2hi(r);
          }
        }
      } else {   // first / last group of the row (clamped byte loads), and NV12 frames (BT.601 on the fly)
#pragma unroll
        for (int c = 0; c < 10; ++c) {
          const int cx = min(max(x0 - 1 + c, 0), W - 1);
          int q0[3], q1[3];
          if (a.format == REGEN_FORMAT_NV12) {
            frame_px(a.frames, REGEN_FORMAT_NV12, f, W, a.H, cx, yl0, q0[0], q0[1], q0[2]);
            frame_px(a.frames, REGEN_FORMAT_NV12, f, W, a.H, cx, yl1, q1[0], q1[1], q1[2]);
          } else {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) { q0[ch] = __ldg(r0 + 3 * cx + ch); q1[ch] = __ldg(r1 + 3 * cx + ch); }
          }
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float p0 = (float)q0[ch], p1 = (float)q1[ch];
            vr[c][ch] = __fmul_rn(fmaf(ly, p1 - p0, p0), 1.0f / 255.0f);
          }
        }
      }
      float dv[9][3];
#pragma unroll
      for (int c = 0; c < 9; ++c)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) dv[c][ch] = __fsub_rn(vr[c + 1][ch], vr[c][ch]);
      // horizontal pass at compile-time phases; edge clamps (x == 0 with d = -1, x == W-1 with d = 0)
      // come out of the clamped column loads (A == B: the lerp returns A exactly)
      float o[G::VALS];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const int ca = q + 1 + Phase<S>::d(j);
          const float lx = Phase<S>::f(j);
          const int e = 3 * (q * S + j);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) o[e + ch] = lx == 0.f ? vr[ca][ch] : fmaf(lx, dv[ca][ch], vr[ca][ch]);
        }
      uint4* st = reinterpret_cast<uint4*>(stage + lane * G::BYTES);
      if (sizeof(TO) == 2) {
#pragma unroll
        for (int k = 0; k < G::CHUNKS; ++k)
          st[k] = make_uint4(pack_bf16(o[8 * k], o[8 * k + 1]), pack_bf16(o[8 * k + 2], o[8 * k + 3]),
                             pack_bf16(o[8 * k + 4], o[8 * k + 5]), pack_bf16(o[8 * k + 6], o[8 * k + 7]));
      } else {
#pragma unroll
        for (int k = 0; k < G::CHUNKS; ++k)
          st[k] = make_uint4(__float_as_uint(o[4 * k]), __float_as_uint(o[4 * k + 1]), __float_as_uint(o[4 * k + 2]),
                             __float_as_uint(o[4 * k + 3]));
      }
    }
    __syncwarp();
    // coalesced copy-out of the warp's run (chunks of groups in owned MBs / past the row are skipped)
    // (fully unrolled: chunk t of a lane sits at a constant offset from the lane's first one)
    uint8_t* drow = (uint8_t*)a.out + (rowi * a.OW + (int64_t)S * 8 * 32 * wc) * 3 * (int64_t)sizeof(TO) + 16 * lane;
    const uint8_t* srow = stage + 16 * lane;
#pragma unroll
    for (int t = 0; t < G::CHUNKS; ++t) {
      const int gl = (lane + 32 * t) / G::CHUNKS;
      if ((amask >> gl) & 1u)
        *reinterpret_cast<uint4*>(drow + 512 * t) = *reinterpret_cast<const uint4*>(srow + 512 * t);
    }
    __syncwarp();
  }
}

// The same pass for u8 frames (D20): integer weights over 2S per axis, so a lane's 8*S HR pixels
// of a row are exact integer sums n = (2S - b)(2S - a) p00 + ... (exact in fp32), each rounded half to
// even once by u8_code (common.cuh). A group is 24*S bytes; chunks of 16 B may straddle the two
// groups of one MB, which share the owned flag.
template <int S>
__global__ void __launch_bounds__(32 * BL_WARPS) bilinear_u8_kernel(ScatterArgs a, int nwc) {
  extern __shared__ __align__(16) uint8_t bsm[];
  constexpr int GB = 24 * S, GW4 = GB / 4;
  constexpr float invD = 1.0f / (float)(4 * S * S);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* stage = bsm + warp * 32 * GB;
  const int W = a.W, W3 = 3 * W, GW = a.GW;
  const int ngroups = W / 8;
  // 32-bit item arithmetic (the host launches this kernel only for < 2^31 items): two 32-bit divisions
  // per item instead of two calls of the 64-bit division routine
  const uint32_t n_items = (uint32_t)((int64_t)a.n_frames * a.OH * nwc);
  for (uint32_t it = blockIdx.x * BL_WARPS + warp; it < n_items; it += gridDim.x * BL_WARPS) {
    const uint32_t rowi32 = it / (uint32_t)nwc;
    const int wc = (int)(it - rowi32 * (uint32_t)nwc);
    const uint32_t f32 = rowi32 / (uint32_t)a.OH;
    const int64_t rowi = rowi32;
    const int Y = (int)(rowi32 - f32 * (uint32_t)a.OH);
    const int64_t f = f32;
    const int g = wc * 32 + lane;
    const int x0 = 8 * g;
    const int my = (Y / S) / 16;
    bool act = g < ngroups;
    if (act) act = __ldg(a.owner + (f * a.GH + my) * GW + x0 / 16) < 0;
    const uint32_t amask = __ballot_sync(0xffffffffu, act);
    if (amask == 0u) continue;
    if (act) {
      const int y = Y / S, i = Y - y * S;
      int yl0 = y + (2 * i + 1 < S ? -1 : 0);
      int bi = 2 * i + 1 < S ? 2 * i + 1 + S : 2 * i + 1 - S;   // ly = bi / (2S)
      if (yl0 < 0) { yl0 = 0; bi = 0; }
      const int yl1 = min(yl0 + 1, a.H - 1);
      if (yl1 == yl0) bi = 0;
      const float b = (float)bi;
      const uint8_t* r0 = a.frames + (f * a.H + yl0) * (int64_t)W3;
      const uint8_t* r1 = a.frames + (f * a.H + yl1) * (int64_t)W3;
      // LR columns x0-1 .. x0+8 (clamped): vertical sums 2S p0 + b (p1 - p0), exact integers in fp32
      float vi[10][3];
      if (W >= 16 && ((((uintptr_t)r0) | ((uintptr_t)r1)) & 3) == 0) {
        uint32_t u0[8], u1[8];
        row_window(r0, x0, W, u0);
        if (bi != 0) {
          row_window(r1, x0, W, u1);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) u1[k] = u0[k];
        }
        float* vf = &vi[0][0];
        const unsigned long long m23 = f2pack(8388608.0f, 8388608.0f), s2 = f2pack(2.0f * S, 2.0f * S);
        const unsigned long long b2 = f2pack(b, b);
#pragma unroll
        for (int e = 0; e < 30; e += 2) {
          const int b0 = 1 + e, b1 = 2 + e;
          const unsigned long long q0 = f2pack(__uint_as_float(__byte_perm(u0[b0 >> 2], 0x4B000000u, 0x7650u | (b0 & 3))),
                                               __uint_as_float(__byte_perm(u0[b1 >> 2], 0x4B000000u, 0x7650u | (b1 & 3))));
          const unsigned long long q1 = f2pack(__uint_as_float(__byte_perm(u1[b0 >> 2], 0x4B000000u, 0x7650u | (b0 & 3))),
                                               __uint_as_float(__byte_perm(u1[b1 >> 2], 0x4B000000u, 0x7650u | (b1 & 3))));
          const unsigned long long p0 = f2sub(q0, m23), p1 = f2sub(q1, m23);
          const unsigned long long r = f2fma(b2, f2sub(p1, p0), f2mul(s2, p0));
          vf[e] = f2lo(r);
          vf[e + 1] = f2hi(r);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 10; ++c) {
          const int cx = min(max(x0 - 1 + c, 0), W - 1);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float p0 = (float)__ldg(r0 + 3 * cx + ch), p1 = (float)__ldg(r1 + 3 * cx + ch);
            vi[c][ch] = fmaf(b, p1 - p0, (float)(2 * S) * p0);
          }
        }
      }
      // horizontal: n = 2S A + num (B - A) (exact), code = rhe(n / (2S)^2) (u8_code); edge clamps
      // come out of the clamped column loads (A == B)
      uint32_t o[GB];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const int ca = q + 1 + Phase<S>::d(j);
          const float n = (float)Phase<S>::num(j);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch)
            o[3 * (q * S + j) + ch] =
                u8_code(fmaf(n, vi[ca + 1][ch] - vi[ca][ch], (float)(2 * S) * vi[ca][ch]), invD);
        }
      uint32_t* st = reinterpret_cast<uint32_t*>(stage + lane * GB);
#pragma unroll
      for (int k = 0; k < GW4; ++k) st[k] = pack_u8x4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
    }
    __syncwarp();
    uint8_t* drow = (uint8_t*)a.out + (rowi * a.OW + (int64_t)S * 8 * 32 * wc) * 3;
    constexpr int NCH = 32 * GB / 16;
#pragma unroll
    for (int t = 0; t < (NCH + 31) / 32; ++t) {
      const int k = lane + 32 * t;
      const int gl = (16 * k) / GB;   // a straddled chunk's two groups share their MB's flag
      if (k < NCH && ((amask >> gl) & 1u))
        *reinterpret_cast<uint4*>(drow + 16 * k) = *reinterpret_cast<const uint4*>(stage + 16 * k);
    }
    __syncwarp();
  }
}

}  // namespace regen

using namespace regen;

namespace regen {

regen_status scatter_launch(const regen_geom& g, const regen_pack_params& p, int scale, const uint8_t* d_frames,
                            const regen_box* d_boxes, const int32_t* d_mb_owner, const void* d_hr_bins, int hr_dtype,
                            void* d_out, int out_dtype, int mode, cudaStream_t s) {
  ScatterArgs a;
  a.frames = d_frames;
  a.format = g.format;
  a.boxes = d_boxes;
  a.owner = d_mb_owner;
  a.hr = d_hr_bins;
  a.out = d_out;
  a.W = g.frame_w;
  a.H = g.frame_h;
  a.OW = g.frame_w * scale;
  a.OH = g.frame_h * scale;
  a.GW = grid_w(g);
  a.GH = grid_h(g);
  a.mb = g.mb;
  a.s = scale;
  a.bin_w = p.bin_w;
  a.bin_h = p.bin_h;
  a.inv_s = 1.0f / (float)scale;
  a.mode = mode;
  a.n_frames = n_frames(g);
  dim3 grid((unsigned)g.frame_h, (unsigned)n_frames(g));
  REGEN_REQUIRE(g.mb == 16, "scatter expects 16-pixel MBs");
  REGEN_REQUIRE(scale == 2 || scale == 3 || scale == 4, "scatter scale must be 2, 3 or 4");
  REGEN_REQUIRE(n_frames(g) <= 65535, "scatter: at most 65535 frames per call");
  const size_t es = out_dtype == REGEN_DTYPE_BF16 ? 2 : (out_dtype == REGEN_DTYPE_U8 ? 1 : 4);
  const size_t cpt = out_dtype == REGEN_DTYPE_U8 ? 4 : 2;   // LR columns per thread of the row kernel
  const size_t npair = ((size_t)g.frame_w + cpt - 1) / cpt;
  const size_t row_words = (npair * 3 * scale * cpt * es / 4 + 3) / 4 * 4;
  const size_t smem = (size_t)g.frame_w * 16 + row_words * 4 + ((size_t)a.GW + 3) / 4 * 16 +
                      3 * (((size_t)g.frame_w * 3 + 15) / 16 * 16) + 16;
  REGEN_REQUIRE(smem <= 200 * 1024, "frame too wide for the scatter kernel (%zu B SMEM)", smem);
  const size_t es_out = es;
  // the warp-per-HR-row bilinear kernel for RGB8 frames; NV12 frames take the row kernel, which converts
  // each LR row once into SMEM for all S HR rows (measured: equal step time to RGB8, where the warp kernel
  // re-converting per HR row cost 5 %)
  const int64_t bl_items = (int64_t)a.n_frames * a.OH * ((g.frame_w / 8 + 31) / 32);
  if (mode == SC_BILINEAR && g.format == REGEN_FORMAT_RGB8 && g.frame_w % 8 == 0 &&
      ((size_t)a.OW * 3 * es_out) % 16 == 0 && bl_items < (1ll << 31) && getenv("REGEN_OLD_BILINEAR") == nullptr) {
    const int ngroups = g.frame_w / 8, nwc = (ngroups + 31) / 32;
    const int64_t items = bl_items;
    const unsigned grid2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + BL_WARPS - 1) / BL_WARPS, 148 * 16));
    auto go2 = [&](auto kern, int bytes) {
      const size_t sm2 = (size_t)BL_WARPS * 32 * bytes;
      if (sm2 > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      REGEN_TRACE("scatter_bilinear", s);
      kern<<<grid2, 32 * BL_WARPS, sm2, s>>>(a, nwc);
    };
    using bf = __nv_bfloat16;
#define BL_GO(S_)                                                                      \
    if (out_dtype == REGEN_DTYPE_BF16) go2(bilinear_kernel<S_, bf>, BL<S_, bf>::BYTES); \
    else if (out_dtype == REGEN_DTYPE_U8) go2(bilinear_u8_kernel<S_>, 24 * S_);         \
    else go2(bilinear_kernel<S_, float>, BL<S_, float>::BYTES);
    if (scale == 2) { BL_GO(2) } else if (scale == 3) { BL_GO(3) } else { BL_GO(4) }
#undef BL_GO
    REGEN_LAUNCH_CHECK();
    return REGEN_OK;
  }
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    REGEN_TRACE(mode == SC_BILINEAR ? "scatter_bilinear" : (mode == SC_OWNED ? "scatter_owned" : "scatter"), s);
    kern<<<grid, SC_THREADS, smem, s>>>(a);
  };
  const bool bf_hr = hr_dtype == REGEN_DTYPE_BF16, bf_out = out_dtype == REGEN_DTYPE_BF16;
  const bool u8_out = out_dtype == REGEN_DTYPE_U8;
  using bf = __nv_bfloat16;
  using u8 = uint8_t;
#define SC_DISPATCH(S_, M_)                                                          \
  if (M_ == SC_BILINEAR) {                                                           \
    if (bf_out) go(scatter_rows_kernel<S_, bf, bf, M_>);                             \
    else if (u8_out) go(scatter_rows_kernel<S_, bf, u8, M_>);                        \
    else go(scatter_rows_kernel<S_, bf, float, M_>);                                 \
  } else if (bf_hr) {                                                                \
    if (bf_out) go(scatter_rows_kernel<S_, bf, bf, M_>);                             \
    else if (u8_out) go(scatter_rows_kernel<S_, bf, u8, M_>);                        \
    else go(scatter_rows_kernel<S_, bf, float, M_>);                                 \
  } else {                                                                           \
    if (bf_out) go(scatter_rows_kernel<S_, float, bf, M_>);                          \
    else if (u8_out) go(scatter_rows_kernel<S_, float, u8, M_>);                     \
    else go(scatter_rows_kernel<S_, float, float, M_>);                              \
  }
#define SC_MODES(S_)                                                                 \
  if (mode == SC_BILINEAR) { SC_DISPATCH(S_, SC_BILINEAR) }                          \
  else if (mode == SC_OWNED) { SC_DISPATCH(S_, SC_OWNED) }                           \
  else { SC_DISPATCH(S_, SC_ALL) }
  REGEN_REQUIRE(mode == SC_ALL || mode == SC_BILINEAR || mode == SC_OWNED, "bad scatter mode");
  REGEN_REQUIRE(mode == SC_BILINEAR || d_hr_bins != nullptr, "scatter: HR bins required");
  if (scale == 2) { SC_MODES(2) } else if (scale == 3) { SC_MODES(3) } else { SC_MODES(4) }
#undef SC_MODES
#undef SC_DISPATCH
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

}  // namespace regen

extern "C" regen_status regen_scatter_blend(const regen_geom* geom, const regen_pack_params* p, int32_t scale,
                                            const uint8_t* d_frames, const regen_box* d_boxes,
                                            const int32_t* d_mb_owner, const void* d_hr_bins, int32_t hr_dtype,
                                            void* d_out, int32_t out_dtype, void* stream) {
  REGEN_NVTX("regen_scatter_blend");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(p != nullptr, "pack params null");
  REGEN_REQUIRE(scale >= 2 && scale <= 4, "scale must be 2, 3 or 4");
  REGEN_REQUIRE(hr_dtype == REGEN_DTYPE_BF16 || hr_dtype == REGEN_DTYPE_FP32, "bad hr dtype");
  REGEN_REQUIRE(out_dtype == REGEN_DTYPE_BF16 || out_dtype == REGEN_DTYPE_FP32 || out_dtype == REGEN_DTYPE_U8,
                "bad out dtype");
  REGEN_REQUIRE(d_frames && d_boxes && d_mb_owner && d_hr_bins && d_out, "null device pointer");
  return scatter_launch(*geom, *p, scale, d_frames, d_boxes, d_mb_owner, d_hr_bins, hr_dtype, d_out, out_dtype, SC_ALL,
                        (cudaStream_t)stream);
}

extern "C" regen_status regen_scatter_bilinear(const regen_geom* geom, int32_t scale, const uint8_t* d_frames,
                                               const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                               void* stream) {
  REGEN_NVTX("regen_scatter_bilinear");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(scale >= 2 && scale <= 4, "scale must be 2, 3 or 4");
  REGEN_REQUIRE(out_dtype == REGEN_DTYPE_BF16 || out_dtype == REGEN_DTYPE_FP32 || out_dtype == REGEN_DTYPE_U8,
                "bad out dtype");
  REGEN_REQUIRE(d_frames && d_mb_owner && d_out, "null device pointer");
  regen_pack_params p;
  memset(&p, 0, sizeof(p));
  return scatter_launch(*geom, p, scale, d_frames, nullptr, d_mb_owner, nullptr, REGEN_DTYPE_BF16, d_out, out_dtype,
                        SC_BILINEAR, (cudaStream_t)stream);
}
