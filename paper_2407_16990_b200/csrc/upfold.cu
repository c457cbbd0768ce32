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
#include <algorithm>
#include <vector>

#include "fold_common.cuh"
#include "net.cuh"
#include "tc_common.cuh"

namespace regen {
using tc::pack_bf16x2;

namespace fold {

// Where the combined HR pixels go. BINS: the HR bin layout [bin][PS*Hr][PS*Wr][4] of
// regen_enhance_packed. FRAME (regen_enhance_scatter): straight into the HR frames
// [S][F][s*H][s*W][3], for owned selected MBs only (the scatter pass writes every other pixel).
struct FrameOut {
  const int32_t* map;        // [bin][bin_h][bin_w] LR bin pixel -> covering box, -1 outside boxes
  const int64_t* dst;        // [bin][bin_h][bin_w] owned pixel: HR frame index of its top-left HR pixel
                             // | rotated << 62; -1: not owned (the scatter pass writes it)
  const regen_box* boxes;
  const int32_t* owner;      // [S][F][GH][GW]
  void* out;
  int out_mode;              // REGEN_DTYPE_*
  int F, W, H, GW, GH, mb, s;
};

template <int PS, bool FRAME>
__global__ void __launch_bounds__(128, 8) combine_kernel(const __nv_bfloat16* P, __nv_bfloat16* out, const uint32_t* mbits,
                                                      const float* bt, const int32_t* num_bins, int Wr, int Hr,
                                                      int res, int bin_w, int bin_h, int c8, FrameOut fo) {
  // grid-stride over the (bin, row) items of the bins actually used (the grid is sized to the GPU)
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_items = *num_bins * Hr;
  if (x >= Wr) return;
  for (int item = blockIdx.y; item < n_items; item += gridDim.y) {
  const int bin = item / Hr, y = item - bin * Hr;
  const int words = (bin_w + 31) / 32;
  const int xl = x / res, yl = y / res;
  // FRAME: only pixels whose source MB is owned by their box (the scatter pass writes the rest)
  int64_t dst = 0;
  bool occ;
  if (FRAME) {
    dst = __ldg(fo.dst + ((size_t)bin * bin_h + yl) * bin_w + xl);
    if (dst < 0) continue;
    occ = true;
  } else {
    occ = (__ldg(mbits + ((size_t)bin * bin_h + yl) * words + xl / 32) >> (xl & 31)) & 1u;
  }
  float acc[PS][PS][3];
  {
    // all partial-sum planes this pixel needs (<= 16 16-B loads over its 3x3 neighbourhood) are
    // issued before any is used, so their latencies overlap
    const size_t pstride = (size_t)Wr * 8;
    constexpr int NL = n_loads(PS);
    uint4 q[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int ny = load_ny(PS, l), nx = load_nx(PS, l), pl = load_pl(PS, l);
      const int yy = y + ny, xx = x + nx;
      q[l] = (!occ || yy < 0 || yy >= Hr || xx < 0 || xx >= Wr)   // zero padding at the bin edge
                 ? make_uint4(0, 0, 0, 0)
                 : __ldg(reinterpret_cast<const uint4*>(P + ((size_t)bin * Hr + yy) * c8 * pstride +
                                                        (size_t)pl * pstride + (size_t)xx * 8));
    }
    accumulate<PS>(q, acc);
  }
  const float b0 = __ldg(bt), b1 = __ldg(bt + 1), b2 = __ldg(bt + 2);
  if (!FRAME) {
    const int WO = Wr * PS;
#pragma unroll
    for (int i = 0; i < PS; ++i) {
      __nv_bfloat16* o = out + (((size_t)bin * Hr * PS + (size_t)y * PS + i) * WO + (size_t)x * PS) * 4;
#pragma unroll
      for (int j = 0; j < PS; ++j) {
        uint2 w;
        w.x = pack_bf16x2(occ ? acc[i][j][0] + b0 : 0.f, occ ? acc[i][j][1] + b1 : 0.f);
        w.y = pack_bf16x2(occ ? acc[i][j][2] + b2 : 0.f, 0.f);
        *reinterpret_cast<uint2*>(o + 4 * j) = w;
      }
    }
  } else {
    store_frame<PS>(acc, b0, b1, b2, dst, res, x, y, fo.W * fo.s, fo.out, fo.out_mode);
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
                                 const int32_t* d_num_bins, int bin_w, int bin_h, cudaStream_t s,
                                 const FoldFrameArgs* fa) {
  const ConvDesc& d = net->convs[net->fold_conv];
  const ConvDesc& up = net->convs[net->fold_conv - 2];
  const ConvDesc& tail = net->convs[net->fold_conv - 1];
  const int p = up.ps, res = d.res;
  const int Wr = bin_w * res, Hr = bin_h * res;
  const int c8 = (d.cout + 7) / 8;
  dim3 grid((unsigned)((Wr + 127) / 128), (unsigned)std::min(max_bins * Hr, 148 * 16));
  const float* bt = net->d_w32 + tail.b_off;
  const __nv_bfloat16* Pb = (const __nv_bfloat16*)P;
  __nv_bfloat16* o = (__nv_bfloat16*)hr_bins;
  fold::FrameOut fo;
  memset(&fo, 0, sizeof(fo));
  if (fa) {
    fo.map = fa->map;
    fo.dst = fa->dst;
    fo.boxes = fa->boxes;
    fo.owner = fa->owner;
    fo.out = fa->out;
    fo.out_mode = fa->out_dtype;
    fo.F = fa->geom.F;
    fo.W = fa->geom.frame_w;
    fo.H = fa->geom.frame_h;
    fo.GW = grid_w(fa->geom);
    fo.GH = grid_h(fa->geom);
    fo.mb = fa->geom.mb;
    fo.s = net->cfg.scale;
  }
  REGEN_TRACE(fa ? "fold_combine_frames" : "fold_combine", s);
#define LAUNCH(PS_, FR_) \
  fold::combine_kernel<PS_, FR_><<<grid, 128, 0, s>>>(Pb, o, mbits, bt, d_num_bins, Wr, Hr, res, bin_w, bin_h, c8, fo)
  if (p == 2) {
    if (fa) LAUNCH(2, true); else LAUNCH(2, false);
  } else if (p == 3) {
    if (fa) LAUNCH(3, true); else LAUNCH(3, false);
  } else {
    REGEN_REQUIRE(false, "fold: unsupported pixel-shuffle factor %d", p);
  }
#undef LAUNCH
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

}  // namespace regen
