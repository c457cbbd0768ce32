// UP∘TAIL fold combine, shared by the standalone combine kernel (upfold.cu) and the fold conv with
// the combine fused into its epilogue (conv_tc.cu, ROLE_FOLDF), so both sum the partials of a pixel
// in exactly the same order (bit-identical results). See upfold.cu for the algebra:
//   out[o](y,x,i,j) = occ(y,x) * ( bt[o] + sum_n P[n,i,j,o](y+ny, x+nx) ).
#pragma once
#include <utility>

#include "net.cuh"
#include "tc_common.cuh"

namespace regen {
namespace fold {

// sub-pixels i of a target whose window reaches neighbour row ny, and their count
__host__ __device__ constexpr int cnt(int ny, int p) { return ny == 0 ? p : 1; }
__host__ __device__ constexpr int first(int ny, int p) { return ny == 1 ? p - 1 : 0; }
// channel offset of neighbour block n = (ny, nx) (raster order over {-1,0,1}^2)
__host__ __device__ constexpr int block_off(int ny, int nx, int p) {
  int off = 0;
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b) {
      if (a == ny && b == nx) return off;
      off += cnt(a, p) * cnt(b, p) * 3;
    }
  return off;
}
__host__ __device__ constexpr int n_channels(int p) { return 3 * (p + 2) * (p + 2); }

// the 16-B plane loads of one pixel's combine, in (neighbour, plane) order: l-th load
__host__ __device__ constexpr int plane_lo(int ny, int nx, int p) { return block_off(ny, nx, p) / 8; }
__host__ __device__ constexpr int plane_hi(int ny, int nx, int p) {
  return (block_off(ny, nx, p) + cnt(ny, p) * cnt(nx, p) * 3 - 1) / 8;
}
__host__ __device__ constexpr int n_loads(int p) {
  int n = 0;
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b) n += plane_hi(a, b, p) - plane_lo(a, b, p) + 1;
  return n;
}
// (ny, nx, plane) of load l, packed as (ny+1)*3 + (nx+1) in the high bits
__host__ __device__ constexpr int load_code(int p, int l) {
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b) {
      const int n = plane_hi(a, b, p) - plane_lo(a, b, p) + 1;
      if (l < n) return ((a + 1) * 3 + (b + 1)) * 64 + plane_lo(a, b, p) + l;
      l -= n;
    }
  return 0;
}
__host__ __device__ constexpr int load_ny(int p, int l) { return load_code(p, l) / 64 / 3 - 1; }
__host__ __device__ constexpr int load_nx(int p, int l) { return load_code(p, l) / 64 % 3 - 1; }
__host__ __device__ constexpr int load_pl(int p, int l) { return load_code(p, l) % 64; }

template <int PS>
__device__ __forceinline__ void acc_zero(float (&acc)[PS][PS][3]) {
#pragma unroll
  for (int i = 0; i < PS; ++i)
#pragma unroll
    for (int j = 0; j < PS; ++j)
#pragma unroll
      for (int o = 0; o < 3; ++o) acc[i][j][o] = 0.f;
}

// add the partials load l (16 B = 8 channels of one plane of neighbour (ny, nx)) carries
template <int PS, int L>
__device__ __forceinline__ void acc_load(const uint4& ql, float (&acc)[PS][PS][3]) {
  constexpr int ny = load_ny(PS, L), nx = load_nx(PS, L), pl = load_pl(PS, L);
  constexpr int off = block_off(ny, nx, PS), ci = cnt(ny, PS), cj = cnt(nx, PS);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&ql);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int ch = pl * 8 + e - off;   // index within the neighbour's block
    if (ch < 0 || ch >= ci * cj * 3) continue;
    const float v = (e & 1) ? __high2float(h[e / 2]) : __low2float(h[e / 2]);
    const int o = ch % 3, t = ch / 3, jj = t % cj, ii = t / cj;
    acc[first(ny, PS) + ii][first(nx, PS) + jj][o] += v;
  }
}

template <int PS, int L = 0>
__device__ __forceinline__ void acc_all(const uint4 (&q)[n_loads(PS)], float (&acc)[PS][PS][3]) {
  if constexpr (L < n_loads(PS)) {
    acc_load<PS, L>(q[L], acc);
    acc_all<PS, L + 1>(q, acc);
  }
}

// acc[i][j][o] = sum of the partials the loads q[] (in load order) carry for sub-pixel (i, j);
// every caller adds in this order (load l ascending, channel ascending): bit-identical results
template <int PS>
__device__ __forceinline__ void accumulate(const uint4 (&q)[n_loads(PS)], float (&acc)[PS][PS][3]) {
  acc_zero<PS>(acc);
  acc_all<PS>(q, acc);
}

// the same sum with the loads issued in batches of B (fewer live registers): ld(l) returns load l
template <int PS, int B, int L0 = 0, typename LD>
__device__ __forceinline__ void accumulate_batched(const LD& ld, float (&acc)[PS][PS][3]) {
  if constexpr (L0 == 0) acc_zero<PS>(acc);
  if constexpr (L0 < n_loads(PS)) {
    constexpr int NB = (n_loads(PS) - L0) < B ? (n_loads(PS) - L0) : B;
    uint4 q[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) q[k] = ld(L0 + k);
    [&]<int... K>(std::integer_sequence<int, K...>) { (acc_load<PS, L0 + K>(q[K], acc), ...); }(
        std::make_integer_sequence<int, NB>{});
    accumulate_batched<PS, B, L0 + NB>(ld, acc);
  }
}

// NE u8 codes (low bytes of q) to o, which is A bytes past a 4-B boundary: a head of 1-3 bytes (u8
// and/or u16), whole 32-bit words, a tail (u16 and/or u8) -- 3 or 4 stores for NE = 9 instead of 9.
template <int NE, int A>
__device__ __forceinline__ void store_codes_at(uint8_t* o, const uint32_t (&q)[NE]) {
  constexpr int H0 = (4 - A) & 3;
  constexpr int H = H0 < NE ? H0 : NE;
  if constexpr (H & 1) o[0] = (uint8_t)q[0];
  if constexpr (H >= 2) *reinterpret_cast<uint16_t*>(o + (H & 1)) = (uint16_t)__byte_perm(q[H & 1], q[(H & 1) + 1], 0x0040);
  constexpr int NW = (NE - H) / 4;
#pragma unroll
  for (int w = 0; w < NW; ++w)
    *reinterpret_cast<uint32_t*>(o + H + 4 * w) = pack_u8x4(q[H + 4 * w], q[H + 4 * w + 1], q[H + 4 * w + 2], q[H + 4 * w + 3]);
  constexpr int T = H + 4 * NW, R = NE - T;
  if constexpr (R >= 2) *reinterpret_cast<uint16_t*>(o + T) = (uint16_t)__byte_perm(q[T], q[T + 1], 0x0040);
  if constexpr (R & 1) o[NE - 1] = (uint8_t)q[NE - 1];
}
template <int NE>
__device__ __forceinline__ void store_codes(uint8_t* o, const uint32_t (&q)[NE]) {
  switch ((uintptr_t)o & 3) {
    case 0: store_codes_at<NE, 0>(o, q); break;
    case 1: store_codes_at<NE, 1>(o, q); break;
    case 2: store_codes_at<NE, 2>(o, q); break;
    default: store_codes_at<NE, 3>(o, q); break;
  }
}

// The PS x PS HR block of one LR bin pixel inside the HR frame (D7 un-rotation: bin-HR sub-pixel
// (i, j) -> frame (j, i) unrotated, (i, PS-1-j) rotated; for res 2 (x4) the block is offset inside
// the LR pixel's 4x4 square by the res-2 sub-position). Values rounded to bf16 first (bit-identical
// to the HR-bin round trip of the separate calls). Each frame row of the block gets 3*PS contiguous
// elements, stored as 32-bit words after a leading 16-bit one when misaligned.
// dst = HR frame index of the LR pixel's top-left HR pixel | rotated << 62.
template <int PS>
__device__ __forceinline__ void store_frame(const float (&acc)[PS][PS][3], float b0, float b1, float b2, int64_t dst,
                                            int res, int x, int y, int OW, void* out, int out_mode) {
  const bool rot = (dst >> 62) & 1;
  int64_t base = dst & ((1ll << 62) - 1);
  if (res > 1) {
    const int sx2 = x % res, sy2 = y % res;
    base += rot ? (int64_t)(PS * (res - 1 - sx2)) * OW + PS * sy2 : (int64_t)(PS * sy2) * OW + PS * sx2;
  }
#pragma unroll
  for (int r = 0; r < PS; ++r) {   // frame row r of the block
    float v[3 * PS];
#pragma unroll
    for (int c = 0; c < PS; ++c) {   // frame column c
      // bin-HR sub-pixel (c, PS-1-r) when rotated, (r, c) otherwise (compile-time indices)
      v[3 * c] = (rot ? acc[c][PS - 1 - r][0] : acc[r][c][0]) + b0;
      v[3 * c + 1] = (rot ? acc[c][PS - 1 - r][1] : acc[r][c][1]) + b1;
      v[3 * c + 2] = (rot ? acc[c][PS - 1 - r][2] : acc[r][c][2]) + b2;
    }
    const size_t e0 = (size_t)(base + (int64_t)r * OW) * 3;   // element index of the run
    if (out_mode == REGEN_DTYPE_U8) {   // D20: quantised from the bf16 value (= the HR-bin round trip)
      constexpr int NE = 3 * PS;
      uint32_t q[NE];
      const __nv_bfloat162 zero = __floats2bfloat162_rn(0.f, 0.f), one = __floats2bfloat162_rn(1.f, 1.f);
#pragma unroll
      for (int e = 0; e < NE; e += 2) {   // bf16x2 round + clamp, then the exact x255 and rounding fma
        const __nv_bfloat162 h = __hmin2(__hmax2(__floats2bfloat162_rn(v[e], e + 1 < NE ? v[e + 1] : 0.f), zero), one);
        q[e] = u8_code(__low2float(h), 255.0f);
        if (e + 1 < NE) q[e + 1] = u8_code(__high2float(h), 255.0f);
      }
      store_codes<NE>((uint8_t*)out + e0, q);
    } else if (out_mode == REGEN_DTYPE_FP32) {
      float* o = (float*)out + e0;
#pragma unroll
      for (int e = 0; e < 3 * PS; ++e) o[e] = __bfloat162float(__float2bfloat16_rn(v[e]));
    } else {
      __nv_bfloat16* o = (__nv_bfloat16*)out + e0;
      constexpr int NE = 3 * PS;
      if (e0 & 1) {   // odd start: one 16-bit store, then 32-bit pairs
        o[0] = __float2bfloat16_rn(v[0]);
#pragma unroll
        for (int e = 1; e + 1 < NE; e += 2) *reinterpret_cast<uint32_t*>(o + e) = tc::pack_bf16x2(v[e], v[e + 1]);
        if ((NE - 1) % 2 == 1) o[NE - 1] = __float2bfloat16_rn(v[NE - 1]);
      } else {
#pragma unroll
        for (int e = 0; e + 1 < NE; e += 2) *reinterpret_cast<uint32_t*>(o + e) = tc::pack_bf16x2(v[e], v[e + 1]);
        if (NE % 2 == 1) o[NE - 1] = __float2bfloat16_rn(v[NE - 1]);
      }
    }
  }
}

}  // namespace fold
}  // namespace regen
