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
  // separable bilinear (D10): the block first interpolates the LR row pair vertically for the LR
  // columns its 8*128 HR pixels touch, into SMEM
  __shared__ float vrow[3 * (8 * 128 / 2 + 4)];
  const int Xb = blockIdx.x * blockDim.x * 8;
  const int xa_blk = min((int)fmaxf(((float)Xb + 0.5f) * a.inv_s - 0.5f, 0.0f), a.W - 1);
  const int xb_blk = min((int)fmaxf(((float)min(Xb + 8 * (int)blockDim.x, a.OW) - 0.5f) * a.inv_s - 0.5f, 0.0f) + 1, a.W - 1);
  {
    const uint8_t* img = a.frames + sf * (int64_t)a.H * a.W * 3;
    const float sy = fmaxf(((float)Y + 0.5f) * a.inv_s - 0.5f, 0.0f);
    const int yl0 = min((int)sy, a.H - 1);
    const int yl1 = min(yl0 + 1, a.H - 1);
    const float ly = sy - (float)yl0;
    const uint8_t* r0 = img + ((size_t)yl0 * a.W + xa_blk) * 3;
    const uint8_t* r1 = img + ((size_t)yl1 * a.W + xa_blk) * 3;
    const int n = (xb_blk - xa_blk + 1) * 3;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const float p0 = (float)r0[i], p1 = (float)r1[i];
      vrow[i] = fmaf(ly, p1 - p0, p0);
    }
  }
  __syncthreads();
  if (X0 >= a.OW) return;
  float o[24];
  // the 8 pixels lie in one MB column (16*s is a multiple of 8), so one owner lookup serves them all
  const int32_t b = a.owner[(sf * a.GH + Y / (a.mb * a.s)) * a.GW + X0 / (a.mb * a.s)];
  if (b >= 0) {
    const regen_box* bp = a.boxes + b;
    const int x0 = bp->x0, y0 = bp->y0, hh = bp->h, bin = bp->bin, bbx = bp->bx, bby = bp->by, rot = bp->rotated;
    const int HW = a.s * a.bin_w, HH = a.s * a.bin_h;
    const int u0 = X0 - a.s * x0, v = Y - a.s * y0;
    const TH* hb = (const TH*)a.hr + (size_t)bin * HH * HW * 4;
    // 8 B per pixel (4 channels); one 8-B load per pixel
    const TH* src = !rot ? hb + ((size_t)(a.s * bby + v) * HW + a.s * bbx + u0) * 4
                         : hb + ((size_t)(a.s * bby + u0) * HW + a.s * bbx + (a.s * hh - 1 - v)) * 4;
    const size_t step = !rot ? 4 : (size_t)HW * 4;   // rotated 90 deg CW: box-local (u, v) <- bin (s*h-1-v, u)
    if (sizeof(TH) == 2) {
      uint2 q[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) q[k] = *reinterpret_cast<const uint2*>(src + (size_t)k * step);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q[k].x));
        const float2 f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q[k].y));
        o[3 * k] = f01.x;
        o[3 * k + 1] = f01.y;
        o[3 * k + 2] = f23.x;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 f = *reinterpret_cast<const float4*>(src + (size_t)k * step);
        o[3 * k] = f.x;
        o[3 * k + 1] = f.y;
        o[3 * k + 2] = f.z;
      }
    }
  } else {
    // horizontal pass over the block's vertically interpolated LR row segment (SMEM)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float sx = fmaxf(((float)(X0 + k) + 0.5f) * a.inv_s - 0.5f, 0.0f);
      const int xl0 = min((int)sx, a.W - 1);
      const int xl1 = min(xl0 + 1, a.W - 1);
      const float lx = sx - (float)xl0;
      const float* v0 = vrow + 3 * (xl0 - xa_blk);
      const float* v1 = vrow + 3 * (xl1 - xa_blk);
#pragma unroll
      for (int c = 0; c < 3; ++c) o[3 * k + c] = fmaf(lx, v1[c] - v0[c], v0[c]) * (1.0f / 255.0f);
    }
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
  REGEN_REQUIRE(scale >= 2 && scale <= 8, "scale must be in [2, 8]");
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
