// Upsampler-tail fold (a7, reading D11; see DESIGN.md §5 "UP∘TAIL fold").
//
// EDSR ends with  UP: conv C -> C*p^2, PixelShuffle(p), occupancy mask   and
//                 TAIL: conv C -> 3 at HR, occupancy mask.
// Nothing non-linear sits between them, so the pair is one linear map from the source-grid features
// f (C channels) to HR RGB. The per-conv mask (D8) is what keeps it from being a plain 5x5 conv: an
// HR neighbour of an output pixel contributes only if the source pixel z it lies in is occupied.
// Decomposing the tail's 3x3 HR window by that source pixel z = target + n (n in {-1,0,1}^2) gives
//
//   out[o](y,x,i,j) = occ(y,x) * ( bt[o] + sum_n P[n,i,j,o](y+ny, x+nx) )
//   P[n,i,j,o](z)  = occ(z) * ( sum_{ci,ky,kx} Wp[n,i,j,o][ci][ky][kx] f[ci](z+k-1) + cp[n,i,j,o] )
//
// where (i,j) is the target's sub-pixel, (n,i,j) runs over the (p+2)^2 pairs whose 3x3 HR window
// reaches into z (ny = -1 only for i = 0, ny = +1 only for i = p-1), and Wp / cp are the tail weights
// contracted with the upsampler's weights / bias (fp64 on the host, from the bf16-rounded weights).
// P is an ordinary masked 3x3 conv C -> 3(p+2)^2 (75 channels at p = 3, 48 at p = 2) that runs on
// the tcgen05 conv kernel (ROLE_FOLD); fold_combine adds the <= 4 partials of every HR pixel. The
// result equals UP -> mask -> TAIL -> mask up to rounding (no bf16 HR activation is formed), at
// 3(p+2)^2 * 9C instead of (p^2 + 3p^2) * 9C multiply-adds per source pixel, and without the
// HR activation round trip through HBM (9.4 MB per 128x128 bin at C = 32, p = 3).
#include <vector>

#include "net.cuh"
#include "tc_common.cuh"

namespace regen {
using tc::pack_bf16x2;

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

template <int PS, typename TO>
__global__ void __launch_bounds__(128) combine_kernel(const __nv_bfloat16* P, TO* out, const uint32_t* mbits,
                                                      const float* bt, const int32_t* num_bins, int Wr, int Hr,
                                                      int res, int bin_w, int bin_h, int c8) {
  const int bin = blockIdx.z;
  if (bin >= *num_bins) return;
  const int y = blockIdx.y;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= Wr) return;
  const int words = (bin_w + 31) / 32;
  const int xl = x / res;
  const bool occ = (__ldg(mbits + ((size_t)bin * bin_h + y / res) * words + xl / 32) >> (xl & 31)) & 1u;
  float acc[PS][PS][3];
#pragma unroll
  for (int i = 0; i < PS; ++i)
#pragma unroll
    for (int j = 0; j < PS; ++j)
#pragma unroll
      for (int o = 0; o < 3; ++o) acc[i][j][o] = 0.f;
  if (occ) {
    const size_t pstride = (size_t)Wr * 8;
#pragma unroll
    for (int ny = -1; ny <= 1; ++ny)
#pragma unroll
      for (int nx = -1; nx <= 1; ++nx) {
        const int yy = y + ny, xx = x + nx;
        if (yy < 0 || yy >= Hr || xx < 0 || xx >= Wr) continue;   // zero padding at the bin edge
        const __nv_bfloat16* base = P + ((size_t)bin * Hr + yy) * c8 * pstride + (size_t)xx * 8;
        constexpr int dummy = 0;
        (void)dummy;
        const int off = block_off(ny, nx, PS), ci = cnt(ny, PS), cj = cnt(nx, PS);
        const int pl0 = off / 8, pl1 = (off + ci * cj * 3 - 1) / 8;
#pragma unroll
        for (int pl = pl0; pl <= pl1; ++pl) {
          const uint4 q = __ldg(reinterpret_cast<const uint4*>(base + (size_t)pl * pstride));
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
          float v[8];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            v[2 * e] = f.x;
            v[2 * e + 1] = f.y;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int ch = pl * 8 + e - off;   // index within the block
            if (ch < 0 || ch >= ci * cj * 3) continue;
            const int o = ch % 3, t = ch / 3, jj = t % cj, ii = t / cj;
            acc[first(ny, PS) + ii][first(nx, PS) + jj][o] += v[e];
          }
        }
      }
  }
  const float b0 = __ldg(bt), b1 = __ldg(bt + 1), b2 = __ldg(bt + 2);
  const int WO = Wr * PS;
#pragma unroll
  for (int i = 0; i < PS; ++i) {
    TO* o = out + (((size_t)bin * Hr * PS + (size_t)y * PS + i) * WO + (size_t)x * PS) * 4;
#pragma unroll
    for (int j = 0; j < PS; ++j) {
      const float r0 = occ ? acc[i][j][0] + b0 : 0.f, r1 = occ ? acc[i][j][1] + b1 : 0.f,
                  r2 = occ ? acc[i][j][2] + b2 : 0.f;
      if (sizeof(TO) == 2) {
        uint2 w;
        w.x = pack_bf16x2(r0, r1);
        w.y = pack_bf16x2(r2, 0.f);
        *reinterpret_cast<uint2*>(o + 4 * j) = w;
      } else {
        *reinterpret_cast<float4*>(o + 4 * j) = make_float4(r0, r1, r2, 0.f);
      }
    }
  }
}

}  // namespace fold

// Append the folded conv (ROLE_FOLD) to the network: weights Wp in the [cout][cin8*8][9] layout of
// w32 and bias cp after it. `w32` holds the (bf16-rounded) weights of every conv already.
void fold_prepare(SRNet* net, std::vector<float>& w32) {
  net->fold_conv = -1;
  const auto& cv = net->convs;
  if (net->cfg.n_resblocks == 0 || cv.size() < 2) return;
  const ConvDesc& up = cv[cv.size() - 2];
  const ConvDesc& tail = cv[cv.size() - 1];
  if (up.role != ROLE_UP || tail.role != ROLE_TAIL) return;
  const int C = net->cfg.channels, p = up.ps, NP = fold::n_channels(p);
  ConvDesc d;
  d.cin = C;
  d.cout = NP;
  d.cin8 = C / 8;
  d.role = ROLE_FOLD;
  d.ps = 1;
  d.res = up.res;
  d.tc_off = 0;
  d.tc_mode = 0;
  std::vector<double> W((size_t)NP * C * 9, 0.0), B(NP, 0.0);
  auto wu = [&](int co, int ci, int k) { return (double)w32[up.w_off + ((size_t)co * up.cin8 * 8 + ci) * 9 + k]; };
  auto wt = [&](int o, int c, int ky, int kx) {
    return (double)w32[tail.w_off + ((size_t)o * tail.cin8 * 8 + c) * 9 + ky * 3 + kx];
  };
  for (int ny = -1; ny <= 1; ++ny)
    for (int nx = -1; nx <= 1; ++nx) {
      const int off = fold::block_off(ny, nx, p), ci_n = fold::cnt(ny, p), cj_n = fold::cnt(nx, p);
      for (int ii = 0; ii < ci_n; ++ii)
        for (int jj = 0; jj < cj_n; ++jj) {
          const int i = fold::first(ny, p) + ii, j = fold::first(nx, p) + jj;
          for (int o = 0; o < 3; ++o) {
            const int ch = off + (ii * cj_n + jj) * 3 + o;
            for (int dy = -1; dy <= 1; ++dy) {
              const int yy = i + dy;                                  // HR row offset within the block
              const int my = yy < 0 ? -1 : (yy >= p ? 1 : 0);
              if (my != ny) continue;
              const int i2 = yy - ny * p;
              for (int dx = -1; dx <= 1; ++dx) {
                const int xx = j + dx;
                const int mx = xx < 0 ? -1 : (xx >= p ? 1 : 0);
                if (mx != nx) continue;
                const int j2 = xx - nx * p;
                for (int c = 0; c < C; ++c) {
                  const double t = wt(o, c, dy + 1, dx + 1);
                  if (t == 0.0) continue;
                  const int cu = c * p * p + i2 * p + j2;
                  B[ch] += t * (double)w32[up.b_off + cu];
                  for (int ci = 0; ci < C; ++ci)
                    for (int k = 0; k < 9; ++k) W[((size_t)ch * C + ci) * 9 + k] += t * wu(cu, ci, k);
                }
              }
            }
          }
        }
    }
  d.w_off = w32.size();
  w32.resize(w32.size() + (size_t)NP * d.cin8 * 8 * 9, 0.0f);
  for (int co = 0; co < NP; ++co)
    for (int ci = 0; ci < C; ++ci)
      for (int k = 0; k < 9; ++k) w32[d.w_off + ((size_t)co * d.cin8 * 8 + ci) * 9 + k] = (float)W[((size_t)co * C + ci) * 9 + k];
  d.b_off = w32.size();
  for (int co = 0; co < NP; ++co) w32.push_back((float)B[co]);
  net->convs.push_back(d);
  net->fold_conv = (int)net->convs.size() - 1;
}

regen_status fold_combine_launch(const SRNet* net, const void* P, void* hr_bins, const uint32_t* mbits, int max_bins,
                                 const int32_t* d_num_bins, int bin_w, int bin_h, cudaStream_t s) {
  const ConvDesc& d = net->convs[net->fold_conv];
  const ConvDesc& up = net->convs[net->fold_conv - 2];
  const ConvDesc& tail = net->convs[net->fold_conv - 1];
  const int p = up.ps, res = d.res;
  const int Wr = bin_w * res, Hr = bin_h * res;
  const int c8 = (d.cout + 7) / 8;
  dim3 grid((unsigned)((Wr + 127) / 128), (unsigned)Hr, (unsigned)max_bins);
  const float* bt = net->d_w32 + tail.b_off;
  const __nv_bfloat16* Pb = (const __nv_bfloat16*)P;
  __nv_bfloat16* o = (__nv_bfloat16*)hr_bins;
  if (p == 2)
    fold::combine_kernel<2, __nv_bfloat16><<<grid, 128, 0, s>>>(Pb, o, mbits, bt, d_num_bins, Wr, Hr, res, bin_w, bin_h, c8);
  else if (p == 3)
    fold::combine_kernel<3, __nv_bfloat16><<<grid, 128, 0, s>>>(Pb, o, mbits, bt, d_num_bins, Wr, Hr, res, bin_w, bin_h, c8);
  else
    REGEN_REQUIRE(false, "fold: unsupported pixel-shuffle factor %d", p);
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

}  // namespace regen
