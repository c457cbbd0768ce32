// Internal helpers shared by the libregen CUDA sources (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <nvtx3/nvToolsExt.h>

#include "../../include/regen.h"

namespace regen {

void set_error(const char* fmt, ...);

#define REGEN_REQUIRE(cond, ...)        \
  do {                                  \
    if (!(cond)) {                      \
      ::regen::set_error(__VA_ARGS__);  \
      return REGEN_E_INVALID;           \
    }                                   \
  } while (0)

#define REGEN_UNSUPPORTED_IF(cond, ...)  \
  do {                                  \
    if (cond) {                         \
      ::regen::set_error(__VA_ARGS__);  \
      return REGEN_E_UNSUPPORTED;       \
    }                                   \
  } while (0)

#define REGEN_CUDA(call)                                                              \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ::regen::set_error("%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return REGEN_E_CUDA;                                                            \
    }                                                                                 \
  } while (0)

#define REGEN_LAUNCH_CHECK()                                                          \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess) {                                                          \
      ::regen::set_error("launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return REGEN_E_CUDA;                                                            \
    }                                                                                 \
  } while (0)

inline int grid_w(const regen_geom& g) { return (g.frame_w + g.mb - 1) / g.mb; }
inline int grid_h(const regen_geom& g) { return (g.frame_h + g.mb - 1) / g.mb; }
inline int words_per_row(const regen_geom& g) { return (grid_w(g) + 31) / 32; }
inline int64_t n_frames(const regen_geom& g) { return (int64_t)g.S * g.F; }
inline int64_t n_mbs(const regen_geom& g) { return n_frames(g) * grid_h(g) * grid_w(g); }

// Workspace carving: sequential 256-B aligned slices.
struct Carver {
  uint8_t* base;
  size_t off = 0;
  explicit Carver(void* b) : base((uint8_t*)b) {}
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    T* p = base ? (T*)(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

regen_status validate_geom(const regen_geom* g);

// Launch tracing (trace.cu, regen_trace_*): when enabled, a TraceScope brackets one kernel launch
// with two CUDA events recorded on its stream; disabled it costs one relaxed load.
bool trace_on();
void trace_begin(const char* name, cudaStream_t s, int* slot);
void trace_end(int slot, cudaStream_t s);
struct TraceScope {
  int slot = -1;
  cudaStream_t s;
  TraceScope(const char* name, cudaStream_t st) : s(st) {
    if (trace_on()) trace_begin(name, st, &slot);
  }
  ~TraceScope() {
    if (slot >= 0) trace_end(slot, s);
  }
};
#define REGEN_TRACE(name, stream) ::regen::TraceScope trace_scope_(name, stream)

// NVTX range around every ABI call (header-only NVTX v3: a no-op unless a tool such as Nsight
// Systems injects itself), so timelines show which call launched which kernels.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define REGEN_NVTX(name) ::regen::NvtxRange nvtx_range_(name)

// ---------------------------------------------------------------- device helpers
// RGB8 of LR pixel (x, y) of frame `frame` (flat stream*F + frame index), from RGB8 or NV12 frames.
// NV12: BT.601 limited range in the 8-bit integer form, nearest chroma (D19; nv12.cu, the oracle).
__device__ __forceinline__ int bt601_clip(int v) { return min(max(v, 0), 255); }
__device__ __forceinline__ void frame_px(const uint8_t* frames, int format, int64_t frame, int W, int H, int x, int y,
                                         int& r, int& g, int& b) {
  if (format == REGEN_FORMAT_NV12) {
    const uint8_t* Y = frames + frame * ((int64_t)W * H * 3 / 2);
    const uint8_t* UV = Y + (int64_t)W * H + (int64_t)(y >> 1) * W + 2 * (x >> 1);
    const int c = 298 * ((int)Y[(int64_t)y * W + x] - 16), d = (int)UV[0] - 128, e = (int)UV[1] - 128;
    r = bt601_clip((c + 409 * e + 128) >> 8);
    g = bt601_clip((c - 100 * d - 208 * e + 128) >> 8);
    b = bt601_clip((c + 516 * d + 128) >> 8);
  } else {
    const uint8_t* p = frames + ((frame * H + y) * (int64_t)W + x) * 3;
    r = p[0];
    g = p[1];
    b = p[2];
  }
}

// D20 u8 output: code = rhe(255 * clamp(v, 0, 1)), exact. With the magic constant 1.5 * 2^23 one
// fma rounds the exact product to the nearest integer, ties to even, into the low mantissa bits:
// u8_code(x, m) = bits(fma(x, m, 1.5 * 2^23)) & 0xff for 0 <= x * m <= 255 exactly representable, or
// whose distance to a .5 tie exceeds fma's rounding error (the callers below state which).
// An enhanced pixel: x = its model-dtype value clamped to [0, 1], m = 255 (bf16 x 255 is exact in
// fp32; an fp32 model value is rounded once, by the fma). A bilinear pixel: x = the exact integer
// sum N of D10's integer weights (over (2s)^2) and codes, m = 1 / (2s)^2: exact for s = 2, 4 (a
// power of two), and for s = 3 no tie exists (every weight numerator is even, 255 v = M / 9) and
// 1/36's rounding moves the product by < 2e-5, far from the nearest .5 (>= 1/18).
constexpr float U8_MAGIC = 12582912.0f;
__device__ __forceinline__ uint32_t u8_code(float x, float m) { return __float_as_uint(fmaf(x, m, U8_MAGIC)); }
// four codes (low bytes) -> one little-endian word
__device__ __forceinline__ uint32_t pack_u8x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
__device__ __forceinline__ uint32_t q_u8(float v) { return u8_code(__saturatef(v), 255.0f) & 0xffu; }

__device__ __forceinline__ uint32_t score_ord(float s) {
  uint32_t b = __float_as_uint(s);
  if (s != s) return 0u;          // NaN lowest
  if (s == 0.0f) b = 0u;          // -0 == +0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t density_ord(double d) {
  uint64_t b = (uint64_t)__double_as_longlong(d);
  if (d != d) return 0ull;
  if (d == 0.0) b = 0ull;
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread (blockDim.x <= 1024, multiple of 32).
// `scratch` must hold 33 ints. Returns exclusive prefix; *total gets the block sum.
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) scratch[lane] = w;  // inclusive warp sums
    if (lane == nw - 1) scratch[32] = w;
  }
  __syncthreads();
  int res = x - v + (warp > 0 ? scratch[warp - 1] : 0);
  *total = scratch[32];
  __syncthreads();
  return res;
}

}  // namespace regen
