// a8: scatter-and-blend, eq. P:461-464 "SR(MB_s) + IN(unselected MBs)", "stitching them
// back to bi-linear-interpolated non-regions". One thread writes 8 consecutive HR pixels (24
// channels) of one output row: either the bilinear value (D10: half-pixel centres, edge clamp,
// fp32) or, inside the HR square of an owned selected MB, the box's HR bin pixel (un-rotated, D7).
// Every HR pixel is written exactly once; stores are 16-B vectors (bf16) / 32-B (fp32).
#include "common.cuh"

namespace regen {

template <typename T>
__device__ __forceinline__ float ld_hr(const T* p);
template <>
__device__ __forceinline__ float ld_hr<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_hr<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

struct ScatterArgs {
  const uint8_t* frames;
  const regen_box* boxes;
  const int32_t* owner;
  const void* hr;
  void* out;
  int W, H, OW, OH, GW, GH, mb, s, bin_w, bin_h;
  float inv_s;
};

template <typename TH, typename TO>
__global__ void __launch_bounds__(128) scatter_kernel(ScatterArgs a) {
  const int64_t sf = blockIdx.z;
  const int Y = blockIdx.y;
  const int X0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (X0 >= a.OW) return;
  const uint8_t* img = a.frames + sf * (int64_t)a.H * a.W * 3;
  // vertical bilinear taps (shared by the 8 pixels)
  float sy = fmaxf(((float)Y + 0.5f) * a.inv_s - 0.5f, 0.0f);
  int y0 = min((int)sy, a.H - 1);
  const int y1 = min(y0 + 1, a.H - 1);
  const float ly = sy - (float)y0;
  const int my = Y / (a.mb * a.s);
  const int32_t* own_row = a.owner + (sf * a.GH + my) * a.GW;
  const int HW = a.s * a.bin_w, HH = a.s * a.bin_h;
  float o[24];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int X = X0 + k;
    float r0 = 0.f, r1 = 0.f, r2 = 0.f;
    if (X < a.OW) {
      const int32_t b = own_row[X / (a.mb * a.s)];
      if (b >= 0) {
        const regen_box bx = a.boxes[b];
        const int u = X - a.s * bx.x0, v = Y - a.s * bx.y0;
        int xb, yb;
        if (bx.rotated) { xb = a.s * bx.bx + (a.s * bx.h - 1 - v); yb = a.s * bx.by + u; }
        else { xb = a.s * bx.bx + u; yb = a.s * bx.by + v; }
        const TH* src = (const TH*)a.hr + (((int64_t)bx.bin * HH + yb) * HW + xb) * 4;
        r0 = ld_hr<TH>(src);
        r1 = ld_hr<TH>(src + 1);
        r2 = ld_hr<TH>(src + 2);
      } else {
        float sx = fmaxf(((float)X + 0.5f) * a.inv_s - 0.5f, 0.0f);
        const int x0 = min((int)sx, a.W - 1);
        const int x1 = min(x0 + 1, a.W - 1);
        const float lx = sx - (float)x0;
        const uint8_t* p00 = img + ((int64_t)y0 * a.W + x0) * 3;
        const uint8_t* p01 = img + ((int64_t)y0 * a.W + x1) * 3;
        const uint8_t* p10 = img + ((int64_t)y1 * a.W + x0) * 3;
        const uint8_t* p11 = img + ((int64_t)y1 * a.W + x1) * 3;
        float v3[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float top = (1.f - lx) * (float)p00[c] + lx * (float)p01[c];
          const float bot = (1.f - lx) * (float)p10[c] + lx * (float)p11[c];
          v3[c] = ((1.f - ly) * top + ly * bot) * (1.0f / 255.0f);
        }
        r0 = v3[0]; r1 = v3[1]; r2 = v3[2];
      }
    }
    o[3 * k] = r0;
    o[3 * k + 1] = r1;
    o[3 * k + 2] = r2;
  }
  TO* dst = (TO*)a.out + ((sf * a.OH + Y) * (int64_t)a.OW + X0) * 3;
  if (X0 + 8 <= a.OW && ((((uintptr_t)dst) & 15) == 0)) {
    if (sizeof(TO) == 2) {
      uint4 v[3];
      uint32_t* w = (uint32_t*)v;
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
        w[i] = *(uint32_t*)&h;
      }
      uint4* d = (uint4*)dst;
      d[0] = v[0]; d[1] = v[1]; d[2] = v[2];
    } else {
      float4* d = (float4*)dst;
#pragma unroll
      for (int i = 0; i < 6; ++i) d[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
    }
  } else {
    for (int k = 0; k < 8 && X0 + k < a.OW; ++k)
      for (int c = 0; c < 3; ++c) {
        if (sizeof(TO) == 2) ((__nv_bfloat16*)dst)[3 * k + c] = __float2bfloat16_rn(o[3 * k + c]);
        else ((float*)dst)[3 * k + c] = o[3 * k + c];
      }
  }
}

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_scatter_blend(const regen_geom* geom, const regen_pack_params* p, int32_t scale,
                                            const uint8_t* d_frames, const regen_box* d_boxes,
                                            const int32_t* d_mb_owner, const void* d_hr_bins, int32_t hr_dtype,
                                            void* d_out, int32_t out_dtype, void* stream) {
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(p != nullptr, "pack params null");
  REGEN_REQUIRE(scale >= 1 && scale <= 8, "bad scale");
  REGEN_REQUIRE(hr_dtype == REGEN_DTYPE_BF16 || hr_dtype == REGEN_DTYPE_FP32, "bad hr dtype");
  REGEN_REQUIRE(out_dtype == REGEN_DTYPE_BF16 || out_dtype == REGEN_DTYPE_FP32, "bad out dtype");
  REGEN_REQUIRE(d_frames && d_boxes && d_mb_owner && d_hr_bins && d_out, "null device pointer");
  const regen_geom g = *geom;
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
  a.bin_w = p->bin_w;
  a.bin_h = p->bin_h;
  a.inv_s = 1.0f / (float)scale;
  dim3 grid((unsigned)((a.OW + 8 * 128 - 1) / (8 * 128)), (unsigned)a.OH, (unsigned)n_frames(g));
  cudaStream_t s = (cudaStream_t)stream;
  if (hr_dtype == REGEN_DTYPE_BF16) {
    if (out_dtype == REGEN_DTYPE_BF16) scatter_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 128, 0, s>>>(a);
    else scatter_kernel<__nv_bfloat16, float><<<grid, 128, 0, s>>>(a);
  } else {
    if (out_dtype == REGEN_DTYPE_BF16) scatter_kernel<float, __nv_bfloat16><<<grid, 128, 0, s>>>(a);
    else scatter_kernel<float, float><<<grid, 128, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}
