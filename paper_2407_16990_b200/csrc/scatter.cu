// a8: scatter-and-blend, eq. P:461-464 "SR(MB_s) + IN(unselected MBs)", "stitching them
// back to bi-linear-interpolated non-regions". Every HR pixel is written exactly once: the bilinear
// value (D10: half-pixel centres, edge clamp, fp32) or, inside the HR square of an owned selected MB,
// the box's HR bin pixel (un-rotated, D7). Stores are 16-B vectors (bf16) / 32-B (fp32).
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
  const int npair = (W + 1) / 2;
  constexpr int WPP = 3 * S * (int)sizeof(TO) / 2;                            // 32-bit words per column pair
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
      for (int x = threadIdx.x; x < W; x += SC_THREADS) {
        float4 v;
        float p0 = (float)r0[3 * x], p1 = (float)r1[3 * x];
        v.x = fmaf(ly, p1 - p0, p0);
        p0 = (float)r0[3 * x + 1]; p1 = (float)r1[3 * x + 1];
        v.y = fmaf(ly, p1 - p0, p0);
        p0 = (float)r0[3 * x + 2]; p1 = (float)r1[3 * x + 2];
        v.z = fmaf(ly, p1 - p0, p0);
        v.w = 0.f;
        vr[x] = v;
      }
    }
    __syncthreads();   // vr ready; previous row's copy-out done
    // ---- 2. horizontal pass: a thread per pair of LR columns -> 2*S HR pixels (6*S values, whole
    // 32-bit words; consecutive threads -> consecutive words: no bank conflicts)
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
          o[e] = fmaf(lx, B.x - A.x, A.x) * (1.0f / 255.0f);
          o[e + 1] = fmaf(lx, B.y - A.y, A.y) * (1.0f / 255.0f);
          o[e + 2] = fmaf(lx, B.z - A.z, A.z) * (1.0f / 255.0f);
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
      if (sizeof(TO) == 2) {
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

}  // namespace regen

using namespace regen;

namespace regen {

regen_status scatter_launch(const regen_geom& g, const regen_pack_params& p, int scale, const uint8_t* d_frames,
                            const regen_box* d_boxes, const int32_t* d_mb_owner, const void* d_hr_bins, int hr_dtype,
                            void* d_out, int out_dtype, int mode, cudaStream_t s) {
  ScatterArgs a;
  a.frames = d_frames;
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
  dim3 grid((unsigned)g.frame_h, (unsigned)n_frames(g));
  REGEN_REQUIRE(g.mb == 16, "scatter expects 16-pixel MBs");
  REGEN_REQUIRE(scale == 2 || scale == 3 || scale == 4, "scatter scale must be 2, 3 or 4");
  REGEN_REQUIRE(n_frames(g) <= 65535, "scatter: at most 65535 frames per call");
  const size_t es = out_dtype == REGEN_DTYPE_BF16 ? 2 : 4;
  const size_t npair = ((size_t)g.frame_w + 1) / 2;
  const size_t row_words = (npair * 3 * scale * es / 2 + 3) / 4 * 4;
  const size_t smem = (size_t)g.frame_w * 16 + row_words * 4 + ((size_t)a.GW + 3) / 4 * 16 +
                      3 * (((size_t)g.frame_w * 3 + 15) / 16 * 16) + 16;
  REGEN_REQUIRE(smem <= 200 * 1024, "frame too wide for the scatter kernel (%zu B SMEM)", smem);
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    REGEN_TRACE(mode == SC_BILINEAR ? "scatter_bilinear" : (mode == SC_OWNED ? "scatter_owned" : "scatter"), s);
    kern<<<grid, SC_THREADS, smem, s>>>(a);
  };
  const bool bf_hr = hr_dtype == REGEN_DTYPE_BF16, bf_out = out_dtype == REGEN_DTYPE_BF16;
  using bf = __nv_bfloat16;
#define SC_DISPATCH(S_, M_)                                                          \
  if (M_ == SC_BILINEAR) {                                                           \
    if (bf_out) go(scatter_rows_kernel<S_, bf, bf, M_>);                             \
    else go(scatter_rows_kernel<S_, bf, float, M_>);                                 \
  } else if (bf_hr) {                                                                \
    if (bf_out) go(scatter_rows_kernel<S_, bf, bf, M_>);                             \
    else go(scatter_rows_kernel<S_, bf, float, M_>);                                 \
  } else {                                                                           \
    if (bf_out) go(scatter_rows_kernel<S_, float, bf, M_>);                          \
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
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(p != nullptr, "pack params null");
  REGEN_REQUIRE(scale >= 2 && scale <= 4, "scale must be 2, 3 or 4");
  REGEN_REQUIRE(hr_dtype == REGEN_DTYPE_BF16 || hr_dtype == REGEN_DTYPE_FP32, "bad hr dtype");
  REGEN_REQUIRE(out_dtype == REGEN_DTYPE_BF16 || out_dtype == REGEN_DTYPE_FP32, "bad out dtype");
  REGEN_REQUIRE(d_frames && d_boxes && d_mb_owner && d_hr_bins && d_out, "null device pointer");
  return scatter_launch(*geom, *p, scale, d_frames, d_boxes, d_mb_owner, d_hr_bins, hr_dtype, d_out, out_dtype, SC_ALL,
                        (cudaStream_t)stream);
}

extern "C" regen_status regen_scatter_bilinear(const regen_geom* geom, int32_t scale, const uint8_t* d_frames,
                                               const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                               void* stream) {
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(scale >= 2 && scale <= 4, "scale must be 2, 3 or 4");
  REGEN_REQUIRE(out_dtype == REGEN_DTYPE_BF16 || out_dtype == REGEN_DTYPE_FP32, "bad out dtype");
  REGEN_REQUIRE(d_frames && d_mb_owner && d_out, "null device pointer");
  regen_pack_params p;
  memset(&p, 0, sizeof(p));
  return scatter_launch(*geom, p, scale, d_frames, nullptr, d_mb_owner, nullptr, REGEN_DTYPE_BF16, d_out, out_dtype,
                        SC_BILINEAR, (cudaStream_t)stream);
}
