// NV12 input. A hardware decoder (the paper's decode stage, §3.1; NVDEC on this
// GPU) hands frames over as NV12: a Y plane [H][W] followed by an interleaved U/V plane [H/2][W/2][2].
// regen_nv12_to_rgb8 converts a call's frames to the RGB8 layout the hot path reads, with the 8-bit
// integer BT.601 limited-range transform (D19):
//   C = Y - 16, D = U - 128, E = V - 128
//   R = clip((298 C + 409 E + 128) >> 8), G = clip((298 C - 100 D - 208 E + 128) >> 8),
//   B = clip((298 C + 516 D + 128) >> 8)
// and nearest (co-sited, replicated) chroma for the 2x2 pixels of each U/V sample. One thread converts
// a 4 x 2 pixel block (two aligned 4-byte Y loads + one 4-byte U/V load, two 12-byte RGB stores). The
// conversion is its own pass on purpose: the bilinear half of the paste-back needs every LR pixel in
// RGB anyway, so fusing it into the gather would not remove it; the 4.5 B per LR pixel it moves (the
// RGB frames of one batch, ~31 MB at 360p x 30, stay L2-resident for the gather and the bilinear pass
// that follow) are < 8% of the step's ~60 B per LR pixel.
#include <algorithm>

#include "common.cuh"

namespace regen {

__device__ __forceinline__ uint32_t clip8(int v) { return (uint32_t)min(max(v, 0), 255); }

__device__ __forceinline__ uint32_t yuv_rgb(int y, int u, int v) {   // r | g << 8 | b << 16
  const int c = 298 * (y - 16), d = u - 128, e = v - 128;
  const uint32_t r = clip8((c + 409 * e + 128) >> 8);
  const uint32_t g = clip8((c - 100 * d - 208 * e + 128) >> 8);
  const uint32_t b = clip8((c + 516 * d + 128) >> 8);
  return r | (g << 8) | (b << 16);
}

// 4 RGB pixels (12 bytes) from 4 Y bytes and 2 U/V pairs
__device__ __forceinline__ uint3 quad_rgb(uint32_t y4, uint32_t uv) {
  const int u0 = uv & 0xFF, v0 = (uv >> 8) & 0xFF, u1 = (uv >> 16) & 0xFF, v1 = uv >> 24;
  const uint32_t p0 = yuv_rgb(y4 & 0xFF, u0, v0), p1 = yuv_rgb((y4 >> 8) & 0xFF, u0, v0);
  const uint32_t p2 = yuv_rgb((y4 >> 16) & 0xFF, u1, v1), p3 = yuv_rgb(y4 >> 24, u1, v1);
  return make_uint3(p0 | (p1 << 24), (p1 >> 8) | (p2 << 16), (p2 >> 16) | (p3 << 8));
}

__global__ void __launch_bounds__(256) nv12_rgb_kernel(const uint8_t* nv12, uint8_t* rgb, int W, int H,
                                                       int64_t n_quads) {
  const int qw = W / 4, qh = H / 2;
  const int64_t frame_in = (int64_t)W * H * 3 / 2, frame_out = (int64_t)W * H * 3;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_quads; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / ((int64_t)qw * qh);
    const int r = (int)(i - f * qw * qh);
    const int qy = r / qw, qx = r - qy * qw;
    const uint8_t* yp = nv12 + f * frame_in;
    const uint8_t* uvp = yp + (int64_t)W * H;
    const uint32_t y0 = *reinterpret_cast<const uint32_t*>(yp + (int64_t)(2 * qy) * W + 4 * qx);
    const uint32_t y1 = *reinterpret_cast<const uint32_t*>(yp + (int64_t)(2 * qy + 1) * W + 4 * qx);
    const uint32_t uv = *reinterpret_cast<const uint32_t*>(uvp + (int64_t)qy * W + 4 * qx);
    uint8_t* o = rgb + f * frame_out + ((int64_t)(2 * qy) * W + 4 * qx) * 3;
    const uint3 a = quad_rgb(y0, uv), b = quad_rgb(y1, uv);
    uint32_t* o0 = reinterpret_cast<uint32_t*>(o);
    uint32_t* o1 = reinterpret_cast<uint32_t*>(o + (int64_t)W * 3);
    o0[0] = a.x; o0[1] = a.y; o0[2] = a.z;
    o1[0] = b.x; o1[1] = b.y; o1[2] = b.z;
  }
}

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_nv12_to_rgb8(const regen_geom* geom, const uint8_t* d_nv12, uint8_t* d_rgb8,
                                           void* stream) {
  REGEN_NVTX("regen_nv12_to_rgb8");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_nv12 && d_rgb8, "null device pointer");
  const regen_geom g = *geom;
  REGEN_REQUIRE(g.frame_w % 4 == 0 && g.frame_h % 2 == 0, "NV12 needs frame_w % 4 == 0 and even frame_h");
  REGEN_REQUIRE(((uintptr_t)d_nv12 & 3) == 0 && ((uintptr_t)d_rgb8 & 3) == 0, "buffers must be 4-byte aligned");
  const int64_t quads = n_frames(g) * (g.frame_w / 4) * (g.frame_h / 2);
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((quads + 255) / 256, 148 * 8));
  REGEN_TRACE("nv12_rgb", s);
  nv12_rgb_kernel<<<grid, 256, 0, s>>>(d_nv12, d_rgb8, g.frame_w, g.frame_h, quads);
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}
