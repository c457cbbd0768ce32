// a6 + a7: stitch the placed boxes into packed bins (§3.3.3) and run the SR network
// over the packed batch (reading D11), with the per-conv occupancy mask that makes every box
// equal to SR of the box alone (reading D8).
//
// paint_kernel   one CTA per placed box writes its index over its bin footprint (the mask map).
// gather_kernel  one thread per bin pixel: covering box -> source pixel (rotation D7) -> u8/255 ->
//                bf16/fp32 chunk of 8 channels (3 real + 5 zero); zero outside boxes.
// conv_simt      fp32 direct 3x3 conv (CUDA cores), the FP32 model path (C1) and the reference
//                path for convs the tcgen05 kernel does not cover; same layout and epilogues.
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include <vector>

#include "net.cuh"

namespace regen {

// ------------------------------------------------------------------------------------ handle

static void build_convs(SRNet* net) {
  const regen_sr_config& c = net->cfg;
  const int C = c.channels, s = c.scale;
  auto add = [&](int cin, int cout, int role, int ps, int res) {
    ConvDesc d;
    d.cin = cin;
    d.cout = cout;
    d.cin8 = (cin + 7) / 8;
    d.role = role;
    d.ps = ps;
    d.res = res;
    d.w_off = d.b_off = d.tc_off = 0;
    d.tc_mode = 0;
    net->convs.push_back(d);
  };
  if (c.n_resblocks == 0) {
    add(3, C, ROLE_TINY0, 1, 1);
    add(C, 3 * s * s, ROLE_TINY1, s, 1);
    return;
  }
  add(3, C, ROLE_HEAD, 1, 1);
  for (int i = 0; i < c.n_resblocks; ++i) {
    add(C, C, ROLE_RES_A, 1, 1);
    add(C, C, ROLE_RES_B, 1, 1);
  }
  add(C, C, ROLE_BODY, 1, 1);
  if (s == 4) {
    add(C, 4 * C, ROLE_UP, 2, 1);
    add(C, 4 * C, ROLE_UP, 2, 2);
  } else {
    add(C, C * s * s, ROLE_UP, s, 1);
  }
  add(C, 3, ROLE_TAIL, 1, s);
}

static uint16_t f32_to_bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float round_bf16_host(float f) {
  uint32_t u = (uint32_t)f32_to_bf16_bits(f) << 16;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

}  // namespace regen

using namespace regen;

namespace regen {
static bool fold_enabled(const SRNet* net, int bin_w);

// The BF16 model runs every conv it executes on the tcgen05 kernels; a configuration with a conv the
// tensor-core kernels do not tile is rejected here (REGEN_E_UNSUPPORTED) instead of silently running
// on a CUDA-core kernel. REGEN_FORCE_SIMT=1 (debug/A-B aid, read at create) is the one explicit way to
// run a BF16 model on the CUDA-core kernel.
static regen_status check_bf16_kernels(const SRNet* net) {
  const char* force = getenv("REGEN_FORCE_SIMT");
  if (force && force[0] == '1') return REGEN_OK;
  const int bw = net->cfg.bin_w, n = net->cfg.n_resblocks;
  REGEN_UNSUPPORTED_IF(!net->use_tc, "BF16 model needs channels %% 16 == 0 (got %d)", net->cfg.channels);
  REGEN_UNSUPPORTED_IF(n == 0, "BF16 tiny model: its C -> 3s^2 conv has no tcgen05 kernel (use FP32)");
  auto planned = [&](size_t i) { return conv_tc_supported(net, net->convs[i], bw); };
  REGEN_UNSUPPORTED_IF(!planned(0), "BF16: no tcgen05 plan for the head conv at bin_w %d", bw);
  if (!resblock_tc_supported(net, bw))
    for (int i = 1; i <= 2 * n; ++i)
      REGEN_UNSUPPORTED_IF(!planned(i), "BF16: no tcgen05 plan for residual conv %d at bin_w %d", i, bw);
  size_t i = 2 * n + 1;
  REGEN_UNSUPPORTED_IF(!planned(i), "BF16: no tcgen05 plan for the body conv at bin_w %d", bw);
  ++i;
  if (net->cfg.scale == 4) {
    REGEN_UNSUPPORTED_IF(!planned(i), "BF16: no tcgen05 plan for the first x2 upsampler at bin_w %d", bw);
    ++i;
  }
  if (!fold_enabled(net, bw)) {
    REGEN_UNSUPPORTED_IF(!planned(i), "BF16: no tcgen05 plan for the upsampler conv at bin_w %d", bw);
    REGEN_UNSUPPORTED_IF(!planned(i + 1), "BF16: no tcgen05 plan for the tail conv at bin_w %d", bw);
  }
  return REGEN_OK;
}
}  // namespace regen

extern "C" regen_status regen_sr_destroy(void* handle);

extern "C" regen_status regen_sr_create(const regen_sr_config* cfg, const float* h_weights, size_t n_weights,
                                        void** out_handle) {
  REGEN_NVTX("regen_sr_create");
  REGEN_REQUIRE(cfg && h_weights && out_handle, "null argument");
  REGEN_REQUIRE(cfg->scale == 2 || cfg->scale == 3 || cfg->scale == 4, "scale must be 2, 3 or 4");
  REGEN_REQUIRE(cfg->channels >= 8 && cfg->channels <= 64 && cfg->channels % 8 == 0,
                "channels must be a multiple of 8 in [8, 64]");
  REGEN_REQUIRE(cfg->n_resblocks >= 0 && cfg->n_resblocks <= 64, "bad n_resblocks");
  REGEN_REQUIRE(cfg->dtype == REGEN_DTYPE_BF16 || cfg->dtype == REGEN_DTYPE_FP32, "bad dtype");
  REGEN_REQUIRE(!(cfg->res_scale != cfg->res_scale), "res_scale is NaN");
  REGEN_REQUIRE(cfg->bin_w >= 4 && cfg->bin_w <= 4096, "bad bin_w %d", cfg->bin_w);
  SRNet* net = new SRNet();
  net->cfg = *cfg;
  {
    auto flag = [](const char* name) { const char* e = getenv(name); return e != nullptr && e[0] == '1'; };
    net->no_fold = flag("REGEN_NO_FOLD");
    net->no_foldf = flag("REGEN_NO_FOLDF");
    net->no_fused_rb = flag("REGEN_NO_FUSED_RESBLOCK");
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&net->n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  build_convs(net);
  size_t need = 0;
  for (auto& d : net->convs) need += (size_t)d.cout * d.cin * 9 + d.cout;
  if (need != n_weights) {
    set_error("n_weights %zu != %zu expected for this config", n_weights, need);
    delete net;
    return REGEN_E_INVALID;
  }
  // fp32 device weights: [cout][cin8*8][9] zero padded, biases after each conv
  std::vector<float> w32;
  size_t src = 0;
  for (auto& d : net->convs) {
    d.w_off = w32.size();
    w32.resize(w32.size() + (size_t)d.cout * d.cin8 * 8 * 9, 0.0f);
    for (int co = 0; co < d.cout; ++co)
      for (int ci = 0; ci < d.cin; ++ci)
        for (int t = 0; t < 9; ++t) {
          float v = h_weights[src + ((size_t)co * d.cin + ci) * 9 + t];
          if (cfg->dtype == REGEN_DTYPE_BF16) v = round_bf16_host(v);
          w32[d.w_off + ((size_t)co * d.cin8 * 8 + ci) * 9 + t] = v;
        }
    src += (size_t)d.cout * d.cin * 9;
    d.b_off = w32.size();
    for (int co = 0; co < d.cout; ++co) w32.push_back(h_weights[src + co]);
    src += d.cout;
  }
  if (cfg->dtype == REGEN_DTYPE_BF16) fold_prepare(net, w32);   // appends the UP∘TAIL fold conv
  cudaError_t e = cudaMalloc(&net->d_w32, w32.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(net->d_w32, w32.data(), w32.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    set_error("weights upload: %s", cudaGetErrorString(e));
    cudaFree(net->d_w32);
    delete net;
    return REGEN_E_CUDA;
  }
  if (cfg->dtype == REGEN_DTYPE_BF16) {
    regen_status st = conv_tc_prepare(net);
    if (st == REGEN_OK && net->use_tc) st = conv_tc_plan_all(net, cfg->bin_w);
    if (st == REGEN_OK && resblock_tc_supported(net, cfg->bin_w)) st = resblock_tc_prepare(net);
    if (st == REGEN_OK) st = check_bf16_kernels(net);
    if (st != REGEN_OK) {
      regen_sr_destroy(net);
      return st;
    }
  }
  *out_handle = net;
  return REGEN_OK;
}

extern "C" regen_status regen_sr_destroy(void* handle) {
  REGEN_NVTX("regen_sr_destroy");
  if (!handle) return REGEN_OK;
  SRNet* net = (SRNet*)handle;
  cudaFree(net->d_w32);
  cudaFree(net->d_wtc);
  conv_tc_release(net);
  resblock_tc_release(net);
  delete net;
  return REGEN_OK;
}

namespace regen {

// ------------------------------------------------------------------------------------ stitch

struct OwnArgs {          // optional: mark bin pixels whose source MB is owned by their box
  const int32_t* owner;  // [S][F][GH][GW], null: skip
  int64_t* dst;
  int F, GH, GW, mb, W, H, s;
  int format;            // REGEN_FORMAT_RGB8 / NV12 of the frames (read by the stitch)
};

// Grids of the stitch kernels are sized to the GPU, not to the capacities (max_boxes, max_bins):
// the counts live on the device, so the kernels loop over them (grid-stride).
constexpr int STITCH_CTAS = 148 * 8;

// map = -1 (and dst = -1) over the bins actually used
__global__ void clear_kernel(const int32_t* num_bins, int max_bins, size_t bin_px, int32_t* map, int64_t* dst) {
  const size_t n = (size_t)min(*num_bins, max_bins) * bin_px;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += stride) {
    reinterpret_cast<int4*>(map)[i] = make_int4(-1, -1, -1, -1);
    if (dst) {
      reinterpret_cast<longlong2*>(dst)[2 * i] = make_longlong2(-1, -1);
      reinterpret_cast<longlong2*>(dst)[2 * i + 1] = make_longlong2(-1, -1);
    }
  }
  for (size_t i = n / 4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    map[i] = -1;
    if (dst) dst[i] = -1;
  }
}

__global__ void paint_kernel(const regen_box* boxes, const int64_t* num_boxes, int64_t max_boxes, int32_t* map,
                             int bin_w, int bin_h, OwnArgs oa) {
  const int64_t nb = min(*num_boxes, max_boxes);
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
  const regen_box bx = boxes[b];
  if (bx.bin < 0) continue;
  const int fw = bx.rotated ? bx.h : bx.w, fh = bx.rotated ? bx.w : bx.h;
  int32_t* m = map + (int64_t)bx.bin * bin_w * bin_h;
  const int32_t* ow = oa.owner ? oa.owner + ((size_t)bx.stream * oa.F + bx.frame) * oa.GH * oa.GW : nullptr;
  for (int i = threadIdx.x; i < fw * fh; i += blockDim.x) {
    const int q = i / fw, p = i - q * fw;
    const size_t px = (size_t)(bx.by + q) * bin_w + bx.bx + p;
    m[px] = (int32_t)b;
    if (ow) {
      const int sx = bx.rotated ? bx.x0 + q : bx.x0 + p;
      const int sy = bx.rotated ? bx.y0 + bx.h - 1 - p : bx.y0 + q;
      const bool own = ow[(sy / oa.mb) * oa.GW + sx / oa.mb] == (int32_t)b;
      const int64_t OW = (int64_t)oa.W * oa.s, OH = (int64_t)oa.H * oa.s;
      const int64_t d = ((((int64_t)bx.stream * oa.F + bx.frame) * OH + (int64_t)oa.s * sy) * OW + (int64_t)oa.s * sx) |
                        ((int64_t)bx.rotated << 62);
      oa.dst[(size_t)bx.bin * bin_w * bin_h + px] = own ? d : -1;
    }
  }
  }
}

template <typename T>
__device__ __forceinline__ T to_t(float v);
template <>
__device__ __forceinline__ float to_t<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_t<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__device__ __forceinline__ float from_t(T v);
template <>
__device__ __forceinline__ float from_t<float>(float v) { return v; }
template <>
__device__ __forceinline__ float from_t<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// LAYOUT 0: activation layout chunk [bin][y][1][x][8]; LAYOUT 1: plain [bin][y][x][4]
template <typename T, int LAYOUT>
__global__ void gather_kernel(const uint8_t* frames, const regen_box* boxes, const int32_t* map,
                              const int32_t* num_bins, int bin_w, int bin_h, int F, int W, int H, T* out,
                              uint32_t* mbits, int format) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_rows = *num_bins * bin_h;
  for (int item = blockIdx.y; item < n_rows; item += gridDim.y) {
  const int b = item / bin_h, y = item - b * bin_h;
  const int32_t id = x < bin_w ? map[((int64_t)b * bin_h + y) * bin_w + x] : -1;
  if (mbits != nullptr) {
    // per-row occupancy bitmask for the tensor-core epilogue: bit x%32 of word [b][y][x/32]
    const uint32_t bits = __ballot_sync(0xffffffffu, id >= 0);
    const int words = (bin_w + 31) / 32;
    if ((threadIdx.x & 31) == 0 && x < bin_w) mbits[((int64_t)b * bin_h + y) * words + x / 32] = bits;
  }
  if (x >= bin_w) continue;
  float v[3] = {0.f, 0.f, 0.f};
  if (id >= 0) {
    const regen_box bx = boxes[id];
    const int p = x - bx.bx, q = y - bx.by;
    const int sx = bx.rotated ? bx.x0 + q : bx.x0 + p;
    const int sy = bx.rotated ? bx.y0 + bx.h - 1 - p : bx.y0 + q;
    int cr, cg, cb;
    frame_px(frames, format, (int64_t)bx.stream * F + bx.frame, W, H, sx, sy, cr, cg, cb);
    v[0] = __fdiv_rn((float)cr, 255.0f);
    v[1] = __fdiv_rn((float)cg, 255.0f);
    v[2] = __fdiv_rn((float)cb, 255.0f);
  }
  if (LAYOUT == 0) {
    T* o = out + (((int64_t)b * bin_h + y) * bin_w + x) * 8;
    if (sizeof(T) == 2) {
      const __nv_bfloat162 h01 = __floats2bfloat162_rn(v[0], v[1]), h2 = __floats2bfloat162_rn(v[2], 0.f);
      *reinterpret_cast<uint4*>(o) = make_uint4(*reinterpret_cast<const uint32_t*>(&h01),
                                                *reinterpret_cast<const uint32_t*>(&h2), 0u, 0u);
    } else {
      reinterpret_cast<float4*>(o)[0] = make_float4(v[0], v[1], v[2], 0.f);
      reinterpret_cast<float4*>(o)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    T* o = out + (((int64_t)b * bin_h + y) * bin_w + x) * 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) o[c] = to_t<T>(c < 3 ? v[c] : 0.0f);
  }
  }
}

// One-pass stitch (bins of width % 32 == 0, <= 1024): per-bin box lists (count, scan, fill), then a
// CTA per band of STITCH_BAND rows of a bin paints the band's box ids into SMEM from its bin's list and
// writes every pixel of the band once: map, the owned-pixel frame destination, the packed input
// (gather, D7 rotation, u8/255 -> bf16/fp32, D9) and the occupancy bits. Replaces clear + paint +
// gather (which wrote map and dst twice and read map back).
constexpr int STITCH_BAND = 8;

__global__ void bin_count_kernel(const regen_box* boxes, const int64_t* num_boxes, int64_t max_boxes, int32_t* cnt) {
  const int64_t nb = min(*num_boxes, max_boxes);
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int bin = boxes[b].bin;
    if (bin >= 0) atomicAdd(cnt + bin, 1);
  }
}

__global__ void __launch_bounds__(1024) bin_scan_kernel(const int32_t* num_bins, int max_bins, int32_t* cnt,
                                                        int32_t* off) {
  __shared__ int scratch[33];
  const int n = min(*num_bins, max_bins);
  int carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int c = i < n ? cnt[i] : 0;
    int tot;
    const int ex = block_exclusive_scan(c, scratch, &tot);
    if (i < n) { off[i] = carry + ex; cnt[i] = carry + ex; }   // cnt becomes the fill cursor
    carry += tot;
  }
  if (threadIdx.x == 0) off[n] = carry;
}

__global__ void bin_fill_kernel(const regen_box* boxes, const int64_t* num_boxes, int64_t max_boxes, int32_t* cur,
                                int32_t* list) {
  const int64_t nb = min(*num_boxes, max_boxes);
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int bin = boxes[b].bin;
    if (bin >= 0) list[atomicAdd(cur + bin, 1)] = (int32_t)b;
  }
}

// the same three steps in one CTA (counts and fill cursors in SMEM): one launch instead of a memset and
// three on the SR stream; a bin's list order is arbitrary (its boxes do not overlap, so the stitch
// paints the same band either way)
__global__ void __launch_bounds__(1024) bin_lists_kernel(const regen_box* boxes, const int64_t* num_boxes,
                                                         int64_t max_boxes, const int32_t* num_bins, int max_bins,
                                                         int32_t* off, int32_t* list) {
  extern __shared__ int32_t bl_cnt[];   // [max_bins + 1]
  __shared__ int scratch[33];
  const int n = min(*num_bins, max_bins);
  const int64_t nbx = min(*num_boxes, max_boxes);
  for (int i = threadIdx.x; i <= n; i += blockDim.x) bl_cnt[i] = 0;
  __syncthreads();
  for (int64_t b = threadIdx.x; b < nbx; b += blockDim.x) {
    const int bin = boxes[b].bin;
    if (bin >= 0 && bin < n) atomicAdd(bl_cnt + bin, 1);
  }
  __syncthreads();
  int carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int c = i < n ? bl_cnt[i] : 0;
    int tot;
    const int ex = block_exclusive_scan(c, scratch, &tot);
    __syncthreads();   // every thread has read its count and the total before the cursors overwrite them
    if (i < n) { off[i] = carry + ex; bl_cnt[i] = carry + ex; }
    carry += tot;
  }
  if (threadIdx.x == 0) off[n] = carry;
  __syncthreads();
  for (int64_t b = threadIdx.x; b < nbx; b += blockDim.x) {
    const int bin = boxes[b].bin;
    if (bin >= 0 && bin < n) list[atomicAdd(bl_cnt + bin, 1)] = (int32_t)b;
  }
}

// A box of the bin being stitched, as the affine map bin pixel (x, y) -> source pixel (sx, sy):
// unrotated sx = ax + x, sy = ay + y; rotated (D7) sx = ax + y, sy = ay - x.
struct StitchBox {
  int32_t id, ax, ay, rot;
  int32_t fr;   // stream * F + frame
};
constexpr int SB_CACHE = 128;   // boxes of one bin kept in SMEM (more: read from the box records)

__device__ __forceinline__ StitchBox stitch_box(const regen_box& bx, int id, int F) {
  StitchBox b;
  b.id = id;
  b.rot = bx.rotated;
  b.ax = bx.rotated ? bx.x0 - bx.by : bx.x0 - bx.bx;
  b.ay = bx.rotated ? bx.y0 + bx.h - 1 + bx.bx : bx.y0 - bx.by;
  b.fr = bx.stream * F + bx.frame;
  return b;
}

template <typename T, int LAYOUT>
__global__ void __launch_bounds__(256, 8) stitch_band_kernel(const uint8_t* frames, const regen_box* boxes,
                                                          const int32_t* off, const int32_t* list,
                                                          const int32_t* num_bins, int max_bins, int bin_w, int bin_h,
                                                          int F, int W, int H, int32_t* map, T* out, uint32_t* mbits,
                                                          OwnArgs oa) {
  // band_ids: -1 empty, 0 .. SB_CACHE-1 the bin-local index of a cached box, SB_CACHE + id otherwise
  extern __shared__ int32_t band_ids[];   // [STITCH_BAND][bin_w]
  __shared__ float u8f[256];              // fp32(u8 / 255), correctly rounded (D9): one table load per value
  __shared__ StitchBox sbox[SB_CACHE];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) u8f[i] = __fdiv_rn((float)i, 255.0f);
  const int nbands = (bin_h + STITCH_BAND - 1) / STITCH_BAND;
  const int items = min(*num_bins, max_bins) * nbands;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int npx = STITCH_BAND * bin_w;
  const int words = bin_w / 32;
  const int64_t OW = (int64_t)oa.W * oa.s, OH = (int64_t)oa.H * oa.s;
  const int64_t gsz = (int64_t)oa.GH * oa.GW;
  const bool mb16 = oa.mb == 16;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int bin = item / nbands, y0 = (item - bin * nbands) * STITCH_BAND;
    const int rows = min(STITCH_BAND, bin_h - y0);
    for (int i = threadIdx.x; i < npx; i += blockDim.x) band_ids[i] = -1;
    __syncthreads();
    // paint: a warp per box of this bin, its footprint rows inside the band; lane 0 caches the box
    const int j0 = off[bin];
    for (int j = j0 + warp; j < off[bin + 1]; j += nwarps) {
      const int id = list[j], loc = j - j0;
      const regen_box& bx = boxes[id];
      if (lane == 0 && loc < SB_CACHE) sbox[loc] = stitch_box(bx, id, F);
      const int tag = loc < SB_CACHE ? loc : SB_CACHE + id;
      const int fw = bx.rotated ? bx.h : bx.w, fh = bx.rotated ? bx.w : bx.h;
      const int ra = max(bx.by, y0), rb = min(bx.by + fh, y0 + rows);
      for (int r = ra; r < rb; ++r)
        for (int p = lane; p < fw; p += 32) band_ids[(r - y0) * bin_w + bx.bx + p] = tag;
    }
    __syncthreads();
    // bin_w dividing the block: a thread keeps its column and steps rows (no division per pixel)
    const int ystep = (blockDim.x % bin_w == 0) ? (int)blockDim.x / bin_w : 0;
    const int xs = threadIdx.x % bin_w, ys = threadIdx.x / bin_w;
    for (int i = threadIdx.x, yy = ys, x = xs; i < rows * bin_w; i += blockDim.x) {
      if (ystep == 0) { yy = i / bin_w; x = i - yy * bin_w; }
      const int y = y0 + yy;
      const int32_t tag = band_ids[i];
      const size_t px = ((size_t)bin * bin_h + y) * bin_w + x;
      if (mbits != nullptr) {   // bin_w % 32 == 0: a warp covers 32 consecutive pixels of one row
        const uint32_t bits = __ballot_sync(0xffffffffu, tag >= 0);
        if (lane == 0) mbits[((size_t)bin * bin_h + y) * words + x / 32] = bits;
      }
      float v[3] = {0.f, 0.f, 0.f};
      int64_t d = -1;
      int32_t id = -1;
      if (tag >= 0) {
        const StitchBox b = tag < SB_CACHE ? sbox[tag] : stitch_box(boxes[tag - SB_CACHE], tag - SB_CACHE, F);
        id = b.id;
        const int sx = b.rot ? b.ax + y : b.ax + x;
        const int sy = b.rot ? b.ay - x : b.ay + y;
        int cr, cg, cb;   // RGB8, or NV12 converted here (D19): the BT.601 conversion fused into the gather
        frame_px(frames, oa.format, b.fr, W, H, sx, sy, cr, cg, cb);
        v[0] = u8f[cr];
        v[1] = u8f[cg];
        v[2] = u8f[cb];
        if (oa.owner) {
          const int mx = mb16 ? sx >> 4 : sx / oa.mb, my = mb16 ? sy >> 4 : sy / oa.mb;
          if (oa.owner[(int64_t)b.fr * gsz + my * oa.GW + mx] == id)
            d = (((int64_t)b.fr * OH + (int64_t)oa.s * sy) * OW + (int64_t)oa.s * sx) | ((int64_t)b.rot << 62);
        }
      }
      map[px] = id;
      if (oa.owner) oa.dst[px] = d;
      if (LAYOUT == 0) {
        T* o = out + px * 8;
        if (sizeof(T) == 2) {
          const __nv_bfloat162 h01 = __floats2bfloat162_rn(v[0], v[1]), h2 = __floats2bfloat162_rn(v[2], 0.f);
          *reinterpret_cast<uint4*>(o) = make_uint4(*reinterpret_cast<const uint32_t*>(&h01),
                                                    *reinterpret_cast<const uint32_t*>(&h2), 0u, 0u);
        } else {
          reinterpret_cast<float4*>(o)[0] = make_float4(v[0], v[1], v[2], 0.f);
          reinterpret_cast<float4*>(o)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      } else {
        T* o = out + px * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = to_t<T>(c < 3 ? v[c] : 0.0f);
      }
      yy += ystep;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------ SIMT conv

struct SimtArgs {
  const void* in;
  void* out;
  const void* skip;
  const float* w;      // [cout][cin8*8][9]
  const float* bias;
  const int32_t* map;  // [bin][bin_h][bin_w] at LR
  const int32_t* num_bins;
  int cin8, cout, role, ps, res;
  int Wr, Hr;          // grid of this conv (bin_w*res, bin_h*res)
  int bin_w, bin_h;
  int out_c8;          // chunks of the output activation (ROLE_UP: cout/ps^2/8)
  float res_scale;
};

template <typename T>
__global__ void __launch_bounds__(128) conv_simt_kernel(SimtArgs a) {
  const int b = blockIdx.z;
  if (b >= *a.num_bins) return;
  const int y = blockIdx.y;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.Wr) return;
  const T* in = (const T*)a.in;
  const int64_t plane = (int64_t)a.Wr * 8;                    // elements per (row, chunk)
  const int64_t rowstride = plane * a.cin8;
  const T* inb = in + (int64_t)b * a.Hr * rowstride;
  const bool occ = a.map[((int64_t)b * a.bin_h + y / a.res) * a.bin_w + x / a.res] >= 0;
  const int K = a.cin8 * 8 * 9;
  for (int co0 = 0; co0 < a.cout; co0 += 16) {
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = (co0 + j < a.cout) ? __ldg(a.bias + co0 + j) : 0.f;
    for (int c8 = 0; c8 < a.cin8; ++c8)
      for (int t = 0; t < 9; ++t) {
        const int yy = y + t / 3 - 1, xx = x + t % 3 - 1;
        if (yy < 0 || xx < 0 || yy >= a.Hr || xx >= a.Wr) continue;
        float v[8];
        const T* src = inb + yy * rowstride + c8 * plane + (int64_t)xx * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = from_t<T>(src[i]);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (co0 + j >= a.cout) break;
          const float* wr = a.w + (int64_t)(co0 + j) * K + (c8 * 8) * 9 + t;
          float s = acc[j];
#pragma unroll
          for (int i = 0; i < 8; ++i) s = fmaf(__ldg(wr + i * 9), v[i], s);
          acc[j] = s;
        }
      }
    // epilogue
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int co = co0 + j;
      if (co >= a.cout) break;
      float v = acc[j];
      if (a.role == ROLE_RES_A || a.role == ROLE_TINY0) v = fmaxf(v, 0.f);
      if (!occ) v = 0.f;
      if (a.role == ROLE_UP || a.role == ROLE_TINY1) {
        const int p2 = a.ps * a.ps;
        const int c = co / p2, i = (co % p2) / a.ps, jj = co % a.ps;
        const int Y = y * a.ps + i, X = x * a.ps + jj;
        const int Wo = a.Wr * a.ps, Ho = a.Hr * a.ps;
        if (a.role == ROLE_UP) {
          T* o = (T*)a.out + (int64_t)b * Ho * (int64_t)Wo * a.out_c8 * 8;
          o[((int64_t)Y * a.out_c8 + c / 8) * Wo * 8 + (int64_t)X * 8 + (c & 7)] = to_t<T>(v);
        } else {
          T* o = (T*)a.out + (int64_t)b * Ho * (int64_t)Wo * 4;
          o[((int64_t)Y * Wo + X) * 4 + c] = to_t<T>(v);
          if (c == 2) o[((int64_t)Y * Wo + X) * 4 + 3] = to_t<T>(0.f);
        }
      } else if (a.role == ROLE_TAIL) {
        T* o = (T*)a.out + ((int64_t)b * a.Hr + y) * (int64_t)a.Wr * 4 + (int64_t)x * 4;
        o[co] = to_t<T>(v);
        if (co == 2) o[3] = to_t<T>(0.f);
      } else {
        const int64_t idx = (int64_t)b * a.Hr * (int64_t)a.Wr * a.out_c8 * 8 +
                            ((int64_t)y * a.out_c8 + co / 8) * a.Wr * 8 + (int64_t)x * 8 + (co & 7);
        if (a.role == ROLE_RES_B) v = occ ? from_t<T>(((const T*)a.skip)[idx]) + a.res_scale * v : 0.f;
        if (a.role == ROLE_BODY) v = occ ? v + from_t<T>(((const T*)a.skip)[idx]) : 0.f;
        ((T*)a.out)[idx] = to_t<T>(v);
      }
    }
  }
}

regen_status conv_simt_launch(const SRNet* net, const ConvDesc& cv, const void* in, void* out, const void* skip,
                              const int32_t* map, int max_bins, const int32_t* d_num_bins, int bin_w, int bin_h,
                              cudaStream_t s) {
  SimtArgs a;
  a.in = in;
  a.out = out;
  a.skip = skip;
  a.w = net->d_w32 + cv.w_off;
  a.bias = net->d_w32 + cv.b_off;
  a.map = map;
  a.num_bins = d_num_bins;
  a.cin8 = cv.cin8;
  a.cout = cv.cout;
  a.role = cv.role;
  a.ps = cv.ps;
  a.res = cv.res;
  a.Wr = bin_w * cv.res;
  a.Hr = bin_h * cv.res;
  a.bin_w = bin_w;
  a.bin_h = bin_h;
  a.out_c8 = cv.role == ROLE_UP ? (cv.cout / (cv.ps * cv.ps) + 7) / 8 : (cv.cout + 7) / 8;
  a.res_scale = net->cfg.res_scale;
  dim3 grid((a.Wr + 127) / 128, a.Hr, max_bins);
  REGEN_TRACE("conv_simt", s);
  if (net->cfg.dtype == REGEN_DTYPE_BF16)
    conv_simt_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(a);
  else
    conv_simt_kernel<float><<<grid, 128, 0, s>>>(a);
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

// ------------------------------------------------------------------------------------ buffers

// frames_out: the buffers of the frame-output calls (regen_enhance_scatter / _owned); with the fused
// fold + combine the HR-resolution partial-sum buffer `u` is never touched and is not carved
EnhanceBufs enhance_bufs(const SRNet* net, const regen_pack_params& p, void* base, bool frames_out, int64_t box_cap) {
  Carver c(base);
  const size_t es = net->cfg.dtype == REGEN_DTYPE_BF16 ? 2 : 4;
  const int C8 = net->cfg.channels / 8, s = net->cfg.scale;
  const size_t px = (size_t)p.max_bins * p.bin_w * p.bin_h;
  EnhanceBufs e;
  e.map = c.take<int32_t>(px);
  e.mbits = c.take<uint32_t>((size_t)p.max_bins * p.bin_h * ((p.bin_w + 31) / 32));
  e.dst = c.take<int64_t>(px);
  e.lists = box_cap > 0 ? c.take<int32_t>(2 * ((size_t)p.max_bins + 1) + (size_t)box_cap) : nullptr;
  e.counters = c.take<int32_t>(N_COUNTERS);
  e.x0 = c.take<uint8_t>(px * 8 * es);
  e.a0 = c.take<uint8_t>(px * C8 * 8 * es);
  if (net->cfg.n_resblocks > 0) {
    e.a1 = c.take<uint8_t>(px * C8 * 8 * es);
    e.a2 = c.take<uint8_t>(px * C8 * 8 * es);
    e.u1 = s == 4 ? (void*)c.take<uint8_t>(px * 4 * C8 * 8 * es) : nullptr;
    const bool fused_fold = frames_out && fold_enabled(net, p.bin_w) && fold_fused_supported(net, p.bin_w);
    e.u = fused_fold ? nullptr : (void*)c.take<uint8_t>(px * s * s * C8 * 8 * es);
  } else {
    e.a1 = e.a2 = e.u1 = e.u = nullptr;
  }
  e.bytes = c.off + 256;
  return e;
}

// `order` alternates along the conv chain: a conv hands out its units in the reverse order of the one
// before it, so it starts on the bins its producer wrote last (still in L2).
// BF16 handles run every conv on tcgen05 (regen_sr_create guarantees a plan for each executed conv);
// FP32 handles (and BF16 under the explicit REGEN_FORCE_SIMT=1 debug switch) on the CUDA-core kernel
static regen_status run_conv(const SRNet* net, const ConvDesc& cv, const void* in, void* out, const void* skip,
                             const EnhanceBufs& e, const regen_pack_params& p, const int32_t* d_num_bins,
                             cudaStream_t s, int order = 0) {
  if (net->use_tc)
    return conv_tc_launch(net, cv, in, out, skip, e.mbits, p.max_bins, d_num_bins, p.bin_w, p.bin_h,
                          e.counters + (&cv - net->convs.data()), s, order & 1);
  return conv_simt_launch(net, cv, in, out, skip, e.map, p.max_bins, d_num_bins, p.bin_w, p.bin_h, s);
}

// the UP∘TAIL fold runs when the folded conv has a tcgen05 plan (REGEN_NO_FOLD=1 forces the literal
// upsampler + tail, for A/B checks)
static bool fold_enabled(const SRNet* net, int bin_w) {
  if (net->fold_conv < 0 || !net->use_tc || net->no_fold) return false;
  return conv_tc_supported(net, net->convs[net->fold_conv], bin_w);
}

static regen_status validate_pack(const regen_pack_params* p, const SRNet* net = nullptr) {
  REGEN_REQUIRE(p != nullptr, "pack params null");
  REGEN_REQUIRE(p->bin_w >= 4 && p->bin_h >= 1 && p->bin_w <= 4096 && p->bin_h <= 4096 && p->max_bins >= 1,
                "bad bin geometry");
  REGEN_REQUIRE(net == nullptr || !net->use_tc || p->bin_w == net->cfg.bin_w,
                "bin_w %d differs from the SR handle's planned bin_w %d", p->bin_w, net ? net->cfg.bin_w : 0);
  return REGEN_OK;
}

}  // namespace regen

namespace regen {

regen_status stitch_into(const regen_geom& g, const regen_pack_params& p, int dtype, int layout,
                         const uint8_t* d_frames, const regen_box* d_boxes, const int64_t* d_num_boxes,
                         int64_t max_boxes, const int32_t* d_num_bins, int32_t* map, void* out, cudaStream_t s,
                         uint32_t* mbits = nullptr, const int32_t* owner = nullptr, int64_t* dst = nullptr,
                         int scale = 0, int32_t* lists = nullptr) {
  OwnArgs oa;
  oa.owner = owner;
  oa.dst = dst;
  oa.W = g.frame_w;
  oa.H = g.frame_h;
  oa.s = scale;
  oa.F = g.F;
  oa.GH = grid_h(g);
  oa.GW = grid_w(g);
  oa.mb = g.mb;
  oa.format = g.format;
  static const bool old_stitch = getenv("REGEN_OLD_STITCH") != nullptr;   // A/B aid: clear + paint + gather
  if (lists != nullptr && p.bin_w % 32 == 0 && p.bin_w <= 1024 && !old_stitch) {
    int32_t* cnt = lists;                       // [max_bins + 1] counts, then fill cursors
    int32_t* off = lists + p.max_bins + 1;      // [max_bins + 1]
    int32_t* list = off + p.max_bins + 1;       // [max_boxes]
    const size_t lsm = sizeof(int32_t) * ((size_t)p.max_bins + 1);
    if (lsm <= 160 * 1024) {
      REGEN_TRACE("stitch_lists", s);
      if (lsm > 48 * 1024) REGEN_CUDA(cudaFuncSetAttribute(bin_lists_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
      bin_lists_kernel<<<1, 1024, lsm, s>>>(d_boxes, d_num_boxes, max_boxes, d_num_bins, p.max_bins, off, list);
    } else {
      const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((max_boxes + 255) / 256, 148 * 4));
      REGEN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)p.max_bins + 1), s));
      REGEN_TRACE("stitch_lists", s);
      bin_count_kernel<<<gb, 256, 0, s>>>(d_boxes, d_num_boxes, max_boxes, cnt);
      bin_scan_kernel<<<1, 1024, 0, s>>>(d_num_bins, p.max_bins, cnt, off);
      bin_fill_kernel<<<gb, 256, 0, s>>>(d_boxes, d_num_boxes, max_boxes, cnt, list);
    }
    REGEN_LAUNCH_CHECK();
    const size_t smem = sizeof(int32_t) * STITCH_BAND * p.bin_w;
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)p.max_bins * ((p.bin_h + STITCH_BAND - 1) / STITCH_BAND),
                                                      148 * 8);
    REGEN_TRACE("stitch", s);
#define STITCH_GO(T, L)                                                                                          \
  stitch_band_kernel<T, L><<<grid, 256, smem, s>>>(d_frames, d_boxes, off, list, d_num_bins, p.max_bins, p.bin_w, \
                                                   p.bin_h, g.F, g.frame_w, g.frame_h, map, (T*)out, mbits, oa)
    if (dtype == REGEN_DTYPE_BF16) {
      if (layout == 0) STITCH_GO(__nv_bfloat16, 0); else STITCH_GO(__nv_bfloat16, 1);
    } else {
      if (layout == 0) STITCH_GO(float, 0); else STITCH_GO(float, 1);
    }
#undef STITCH_GO
    REGEN_LAUNCH_CHECK();
    return REGEN_OK;
  }
  {
    REGEN_TRACE("clear", s);
    clear_kernel<<<STITCH_CTAS, 256, 0, s>>>(d_num_bins, p.max_bins, (size_t)p.bin_w * p.bin_h, map,
                                             owner ? dst : nullptr);
  }
  {
    REGEN_TRACE("paint", s);
    paint_kernel<<<(unsigned)std::min<int64_t>(max_boxes, STITCH_CTAS), 256, 0, s>>>(d_boxes, d_num_boxes, max_boxes,
                                                                                    map, p.bin_w, p.bin_h, oa);
  }
  REGEN_LAUNCH_CHECK();
  dim3 grid((p.bin_w + 127) / 128, (unsigned)std::min<int64_t>((int64_t)p.max_bins * p.bin_h, STITCH_CTAS));
  REGEN_TRACE("gather", s);
  if (dtype == REGEN_DTYPE_BF16) {
    if (layout == 0)
      gather_kernel<__nv_bfloat16, 0><<<grid, 128, 0, s>>>(d_frames, d_boxes, map, d_num_bins, p.bin_w, p.bin_h, g.F,
                                                           g.frame_w, g.frame_h, (__nv_bfloat16*)out, mbits, g.format);
    else
      gather_kernel<__nv_bfloat16, 1><<<grid, 128, 0, s>>>(d_frames, d_boxes, map, d_num_bins, p.bin_w, p.bin_h, g.F,
                                                           g.frame_w, g.frame_h, (__nv_bfloat16*)out, mbits, g.format);
  } else {
    if (layout == 0)
      gather_kernel<float, 0><<<grid, 128, 0, s>>>(d_frames, d_boxes, map, d_num_bins, p.bin_w, p.bin_h, g.F,
                                                   g.frame_w, g.frame_h, (float*)out, mbits, g.format);
    else
      gather_kernel<float, 1><<<grid, 128, 0, s>>>(d_frames, d_boxes, map, d_num_bins, p.bin_w, p.bin_h, g.F,
                                                   g.frame_w, g.frame_h, (float*)out, mbits, g.format);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_stitch_bins(const regen_geom* geom, const regen_pack_params* p, int32_t dtype,
                                          const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                          const int64_t* d_num_boxes, const int32_t* d_num_bins, void* d_lr_bins,
                                          void* d_ws, size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_stitch_bins");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  st = validate_pack(p);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(dtype == REGEN_DTYPE_BF16 || dtype == REGEN_DTYPE_FP32, "bad dtype");
  REGEN_REQUIRE(d_frames && d_boxes && d_num_boxes && d_num_bins && d_lr_bins, "null device pointer");
  REGEN_REQUIRE(max_boxes >= 1 && max_boxes < (1ll << 31), "bad max_boxes");
  const size_t need = (size_t)p->max_bins * p->bin_w * p->bin_h * 4 + 256;
  REGEN_REQUIRE(d_ws && ws_bytes >= need, "workspace too small");
  return stitch_into(*geom, *p, dtype, 1, d_frames, d_boxes, d_num_boxes, max_boxes, d_num_bins, (int32_t*)d_ws,
                     d_lr_bins, (cudaStream_t)stream);
}

extern "C" regen_status regen_enhance_kernel_count(const void* sr, const regen_pack_params* p, int32_t* count) {
  REGEN_REQUIRE(sr && p && count, "null argument");
  const SRNet* net = (const SRNet*)sr;
  const int nr = net->cfg.n_resblocks;
  int n = 3;   // clear + paint + gather
  if (nr == 0) {
    n += 2;
  } else {
    n += 1 + (resblock_tc_supported(net, p->bin_w) ? nr : 2 * nr) + 1;   // head, residual blocks, body
    if (net->cfg.scale == 4) n += 1;                                      // first x2 stage
    n += 2;                                                               // UP + TAIL, or FOLD + combine
  }
  *count = n;
  return REGEN_OK;
}

namespace regen {

// stitch + SR of the packed batch; the HR result goes to hr_bins, or (fa != null, fold path only)
// straight into the HR frames for owned MBs
// partials_only (fold path, fa != null): stop after the fold conv, its partial sums left in e.u for a
// later regen_fold_combine_frames
static regen_status enhance_run(const SRNet* net, const regen_geom* geom, const regen_pack_params* p,
                                const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                const int64_t* d_num_boxes, const int32_t* d_num_bins, void* d_hr_bins,
                                const EnhanceBufs& e, cudaStream_t s, FoldFrameArgs* fa, bool partials_only = false) {
  REGEN_CUDA(cudaMemsetAsync(e.counters, 0, N_COUNTERS * sizeof(int32_t), s));
  regen_status st = stitch_into(*geom, *p, net->cfg.dtype, 0, d_frames, d_boxes, d_num_boxes, max_boxes, d_num_bins,
                                e.map, e.x0, s, e.mbits, fa ? fa->owner : nullptr, e.dst,
                                net->cfg.scale, e.lists);
  if (st != REGEN_OK) return st;
  const auto& cv = net->convs;
  if (net->cfg.n_resblocks == 0) {
    st = run_conv(net, cv[0], e.x0, e.a0, nullptr, e, *p, d_num_bins, s);
    if (st == REGEN_OK) st = run_conv(net, cv[1], e.a0, d_hr_bins, nullptr, e, *p, d_num_bins, s);
    return st;
  }
  size_t i = 0;
  int ord = 0;   // unit order of the next conv launch (alternating, see run_conv)
  st = run_conv(net, cv[i++], e.x0, e.a0, nullptr, e, *p, d_num_bins, s, ord++);     // head -> h
  const void* r = e.a0;
  void* body_out = e.a2;
  if (resblock_tc_supported(net, p->bin_w)) {
    // fused residual blocks (t stays in SMEM), ping-pong a1 <-> a2
    for (int k = 0; k < net->cfg.n_resblocks && st == REGEN_OK; ++k) {
      void* o = (k & 1) ? e.a2 : e.a1;
      st = resblock_tc_launch(net, k, r, o, e.mbits, p->max_bins, d_num_bins, p->bin_w, p->bin_h,
                              e.counters + RB_COUNTER0 + k, s, (ord++) & 1);
      r = o;
      i += 2;
    }
    body_out = (r == e.a1) ? e.a2 : e.a1;
  } else {
    for (int k = 0; k < net->cfg.n_resblocks && st == REGEN_OK; ++k) {
      st = run_conv(net, cv[i++], r, e.a2, nullptr, e, *p, d_num_bins, s, ord++);      // t = relu(conv(r))
      if (st != REGEN_OK) break;
      st = run_conv(net, cv[i++], e.a2, e.a1, r, e, *p, d_num_bins, s, ord++);         // r' = r + s*conv(t)
      r = e.a1;
    }
  }
  if (st == REGEN_OK) st = run_conv(net, cv[i++], r, body_out, e.a0, e, *p, d_num_bins, s, ord++);  // body + h
  if (st != REGEN_OK) return st;
  const void* up_in = body_out;
  if (net->cfg.scale == 4) {   // first x2 stage
    st = run_conv(net, cv[i++], body_out, e.u1, nullptr, e, *p, d_num_bins, s, ord++);
    up_in = e.u1;
  }
  if (st != REGEN_OK) return st;
  if (fold_enabled(net, p->bin_w)) {
    if (fa) {
      fa->map = e.map;
      fa->dst = e.dst;
      if (!partials_only && fold_fused_supported(net, p->bin_w))   // combine fused into the fold conv: no partials in HBM
        return fold_fused_launch(net, up_in, e.mbits, p->max_bins, d_num_bins, p->bin_w, p->bin_h,
                                 e.counters + net->fold_conv, s, (ord++) & 1, *fa);
    }
    // last upsampler + tail as the folded conv (partials in e.u) and the partial-sum combine
    st = run_conv(net, cv[net->fold_conv], up_in, e.u, nullptr, e, *p, d_num_bins, s, ord++);
    if (st == REGEN_OK && !partials_only)
      st = fold_combine_launch(net, e.u, d_hr_bins, e.mbits, p->max_bins, d_num_bins, p->bin_w, p->bin_h, s, fa);
    return st;
  }
  REGEN_REQUIRE(fa == nullptr, "frame output needs the fold path");
  st = run_conv(net, cv[i++], up_in, e.u, nullptr, e, *p, d_num_bins, s, ord++);
  if (st == REGEN_OK) st = run_conv(net, cv[i++], e.u, d_hr_bins, nullptr, e, *p, d_num_bins, s, ord++);  // tail
  return st;
}

static size_t hr_bins_bytes(const SRNet* net, const regen_pack_params& p) {
  const size_t es = net->cfg.dtype == REGEN_DTYPE_BF16 ? 2 : 4;
  const size_t s = (size_t)net->cfg.scale;
  return (size_t)p.max_bins * s * s * p.bin_w * p.bin_h * 4 * es;
}

// workspace of regen_enhance_scatter: the enhance buffers, plus the HR bins when the fold is off
size_t enhance_scatter_ws_bytes(const SRNet* net, const regen_pack_params& p, int64_t box_cap) {
  const size_t e = (enhance_bufs(net, p, nullptr, true, box_cap).bytes + 255) / 256 * 256;
  return fold_enabled(net, p.bin_w) ? e : e + hr_bins_bytes(net, p) + 256;
}

}  // namespace regen

extern "C" regen_status regen_enhance_packed(void* sr, const regen_geom* geom, const regen_pack_params* p,
                                             const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                             const int64_t* d_num_boxes, const int32_t* d_num_bins, void* d_hr_bins,
                                             int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_enhance_packed");
  REGEN_REQUIRE(sr != nullptr, "null SR handle");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  st = validate_pack(p);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_frames && d_boxes && d_num_boxes && d_num_bins && d_hr_bins && d_status, "null device pointer");
  REGEN_REQUIRE(max_boxes >= 1 && max_boxes < (1ll << 31), "bad max_boxes");
  const SRNet* net = (const SRNet*)sr;
  st = validate_pack(p, net);
  if (st != REGEN_OK) return st;
  EnhanceBufs e = enhance_bufs(net, *p, nullptr, false, n_mbs(*geom));
  REGEN_REQUIRE(d_ws && ws_bytes >= e.bytes, "workspace too small (%zu < %zu)", ws_bytes, e.bytes);
  e = enhance_bufs(net, *p, d_ws, false, n_mbs(*geom));
  return enhance_run(net, geom, p, d_frames, d_boxes, max_boxes, d_num_boxes, d_num_bins, d_hr_bins, e,
                     (cudaStream_t)stream, nullptr);
}

namespace regen {
// parts: 1 = the owned MBs' SR pixels, 2 = the bilinear pixels (the rest), 3 = the whole HR frames
static regen_status enhance_scatter_parts(void* sr, const regen_geom* geom, const regen_pack_params* p,
                                          const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                          const int64_t* d_num_boxes, const int32_t* d_num_bins,
                                          const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                          int32_t* d_status, void* d_ws, size_t ws_bytes, cudaStream_t s, int parts) {
  REGEN_REQUIRE(sr != nullptr, "null SR handle");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  st = validate_pack(p);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_frames && d_boxes && d_num_boxes && d_num_bins && d_mb_owner && d_out && d_status,
                "null device pointer");
  REGEN_REQUIRE(max_boxes >= 1 && max_boxes < (1ll << 31), "bad max_boxes");
  REGEN_REQUIRE(out_dtype == REGEN_DTYPE_BF16 || out_dtype == REGEN_DTYPE_FP32 || out_dtype == REGEN_DTYPE_U8,
                "bad out dtype");
  const SRNet* net = (const SRNet*)sr;
  st = validate_pack(p, net);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(net->cfg.scale >= 2, "scale must be >= 2");
  const size_t need = enhance_scatter_ws_bytes(net, *p, n_mbs(*geom));
  REGEN_REQUIRE(d_ws && ws_bytes >= need, "workspace too small (%zu < %zu)", ws_bytes, need);
  EnhanceBufs e = enhance_bufs(net, *p, d_ws, true, n_mbs(*geom));
  if (fold_enabled(net, p->bin_w)) {
    FoldFrameArgs fa;
    fa.geom = *geom;
    fa.map = nullptr;
    fa.boxes = d_boxes;
    fa.owner = d_mb_owner;
    fa.out = d_out;
    fa.out_dtype = out_dtype;
    st = enhance_run(net, geom, p, d_frames, d_boxes, max_boxes, d_num_boxes, d_num_bins, nullptr, e, s, &fa);
    if (st != REGEN_OK || !(parts & 2)) return st;
    return scatter_launch(*geom, *p, net->cfg.scale, d_frames, d_boxes, d_mb_owner, nullptr, net->cfg.dtype, d_out,
                          out_dtype, 1, s);
  }
  void* hr = (uint8_t*)d_ws + (e.bytes + 255) / 256 * 256;
  st = enhance_run(net, geom, p, d_frames, d_boxes, max_boxes, d_num_boxes, d_num_bins, hr, e, s, nullptr);
  if (st != REGEN_OK) return st;
  return scatter_launch(*geom, *p, net->cfg.scale, d_frames, d_boxes, d_mb_owner, hr, net->cfg.dtype, d_out, out_dtype,
                        parts == 3 ? 0 : 2, s);
}
}  // namespace regen

extern "C" regen_status regen_enhance_scatter(void* sr, const regen_geom* geom, const regen_pack_params* p,
                                              const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                              const int64_t* d_num_boxes, const int32_t* d_num_bins,
                                              const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                              int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_enhance_scatter");
  return enhance_scatter_parts(sr, geom, p, d_frames, d_boxes, max_boxes, d_num_boxes, d_num_bins, d_mb_owner, d_out,
                               out_dtype, d_status, d_ws, ws_bytes, (cudaStream_t)stream, 3);
}

extern "C" regen_status regen_enhance_owned(void* sr, const regen_geom* geom, const regen_pack_params* p,
                                            const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                            const int64_t* d_num_boxes, const int32_t* d_num_bins,
                                            const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                            int32_t* d_status, void* d_ws, size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_enhance_owned");
  return enhance_scatter_parts(sr, geom, p, d_frames, d_boxes, max_boxes, d_num_boxes, d_num_bins, d_mb_owner, d_out,
                               out_dtype, d_status, d_ws, ws_bytes, (cudaStream_t)stream, 1);
}

// The SR of regen_enhance_owned split in two stream-ordered halves (fold path only): the convolutions
// up to the UP∘TAIL fold's partial sums (kept in the workspace), and the partial-sum combine that writes
// the owned MBs' HR pixels into the frames. Together bit-identical to regen_enhance_owned; the combine
// can then run on another stream beside the next batch's convolutions.
extern "C" regen_status regen_enhance_partials(void* sr, const regen_geom* geom, const regen_pack_params* p,
                                               const uint8_t* d_frames, const regen_box* d_boxes, int64_t max_boxes,
                                               const int64_t* d_num_boxes, const int32_t* d_num_bins,
                                               const int32_t* d_mb_owner, int32_t* d_status, void* d_ws,
                                               size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_enhance_partials");
  REGEN_REQUIRE(sr != nullptr, "null SR handle");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  const SRNet* net = (const SRNet*)sr;
  st = validate_pack(p, net);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_frames && d_boxes && d_num_boxes && d_num_bins && d_mb_owner && d_status, "null device pointer");
  REGEN_REQUIRE(max_boxes >= 1 && max_boxes < (1ll << 31), "bad max_boxes");
  REGEN_UNSUPPORTED_IF(!fold_enabled(net, p->bin_w), "enhance_partials needs the UP-TAIL fold (BF16 tensor-core path)");
  EnhanceBufs e = enhance_bufs(net, *p, nullptr, false, n_mbs(*geom));
  REGEN_REQUIRE(d_ws && ws_bytes >= e.bytes, "workspace too small (%zu < %zu)", ws_bytes, e.bytes);
  e = enhance_bufs(net, *p, d_ws, false, n_mbs(*geom));
  FoldFrameArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.geom = *geom;
  fa.boxes = d_boxes;
  fa.owner = d_mb_owner;
  return enhance_run(net, geom, p, d_frames, d_boxes, max_boxes, d_num_boxes, d_num_bins, nullptr, e,
                     (cudaStream_t)stream, &fa, true);
}

extern "C" regen_status regen_fold_combine_frames(void* sr, const regen_geom* geom, const regen_pack_params* p,
                                                  const regen_box* d_boxes, const int32_t* d_num_bins,
                                                  const int32_t* d_mb_owner, void* d_out, int32_t out_dtype,
                                                  void* d_ws, size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_fold_combine_frames");
  REGEN_REQUIRE(sr != nullptr, "null SR handle");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  const SRNet* net = (const SRNet*)sr;
  st = validate_pack(p, net);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_boxes && d_num_bins && d_mb_owner && d_out, "null device pointer");
  REGEN_REQUIRE(out_dtype == REGEN_DTYPE_BF16 || out_dtype == REGEN_DTYPE_FP32 || out_dtype == REGEN_DTYPE_U8,
                "bad out dtype");
  REGEN_UNSUPPORTED_IF(!fold_enabled(net, p->bin_w), "fold_combine_frames needs the UP-TAIL fold");
  EnhanceBufs e = enhance_bufs(net, *p, nullptr, false, n_mbs(*geom));
  REGEN_REQUIRE(d_ws && ws_bytes >= e.bytes, "workspace too small (%zu < %zu)", ws_bytes, e.bytes);
  e = enhance_bufs(net, *p, d_ws, false, n_mbs(*geom));
  FoldFrameArgs fa;
  fa.geom = *geom;
  fa.map = e.map;
  fa.dst = e.dst;
  fa.boxes = d_boxes;
  fa.owner = d_mb_owner;
  fa.out = d_out;
  fa.out_dtype = out_dtype;
  return fold_combine_launch(net, e.u, nullptr, e.mbits, p->max_bins, d_num_bins, p->bin_w, p->bin_h,
                             (cudaStream_t)stream, &fa);
}
