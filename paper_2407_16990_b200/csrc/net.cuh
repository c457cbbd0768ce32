// SR network handle and activation layout (internal).
//
// Activation layout (both dtypes): [bin][row][C/8][col][8] — per bin row, C/8 planes of 8-channel
// 16-B (bf16) / 32-B (fp32) chunks, each plane `width` pixels long. One bin row of one plane is a
// contiguous run, so a tcgen05 K-major no-swizzle operand tile (8 rows x 16 B core matrices, rows
// contiguous) is a plain 16-B-aligned slice of it and every 3x3 tap is a start-address offset.
#pragma once
#include <vector>

#include "common.cuh"

namespace regen {

enum ConvRole : int {
  ROLE_HEAD = 0,     // x0 -> h (also the residual stream)
  ROLE_RES_A = 1,    // r -> t = relu(conv)
  ROLE_RES_B = 2,    // t -> r' = r + res_scale * conv
  ROLE_BODY = 3,     // r -> conv + h
  ROLE_UP = 4,       // -> conv, PixelShuffle(ps) into the next resolution
  ROLE_TAIL = 5,     // -> HR output [bin][y][x][4]
  ROLE_TINY0 = 6,    // x0 -> relu(conv)
  ROLE_TINY1 = 7,    // -> conv, PixelShuffle(scale) into the HR output
  ROLE_FOLD = 8,     // UP∘TAIL fold: conv C -> 3(p+2)^2 partial sums (upfold.cu)
  ROLE_FOLDF = 9     // launch variant of ROLE_FOLD with the partial-sum combine fused into the epilogue:
                     // writes the owned MBs' HR pixels straight into the frames (conv_tc.cu)
};

struct ConvDesc {
  int cin, cout;       // real channel counts
  int cin8;            // input chunks of 8 channels
  int role;
  int ps;              // pixel-shuffle factor for ROLE_UP / ROLE_TINY1
  int res;             // resolution factor of the conv's input/output grid relative to LR (1, 2, 3, 4)
  size_t w_off;        // offset (floats) into d_w32: [cout][cin8*8][9] zero padded
  size_t b_off;        // offset (floats) of bias[cout]
  size_t tc_off;       // offset (bytes) into d_wtc (tcgen05 packed bf16 B operand), see conv_tc.cu
  int tc_mode;         // tcgen05 mapping (0 = none)
};

struct SRNet {
  regen_sr_config cfg;
  std::vector<ConvDesc> convs;
  float* d_w32 = nullptr;      // fp32 weights (bf16-rounded for the BF16 model) + biases
  uint8_t* d_wtc = nullptr;    // tcgen05 B-operand images
  size_t wtc_bytes = 0;
  bool use_tc = false;
  void* tc_plans = nullptr;   // tc::NetPlans (conv_tc.cu)
  std::vector<float> tc_weights;   // host copy of the (rounded) weights for B-image packing
  int tc_bin_w = -1;             // bin width the B images were planned for
  void* rb_images = nullptr;     // fused-resblock B images (resblock_tc.cu)
  int fold_conv = -1;            // index of the ROLE_FOLD conv in convs (-1: none)
  int n_sm = 148;                // SMs of the device the handle was created on (persistent grids)
  // A/B switches, read from the environment once by regen_sr_create (REGEN_NO_FOLD, REGEN_NO_FOLDF,
  // REGEN_NO_FUSED_RESBLOCK): measurement aids, every default is the fastest path
  bool no_fold = false, no_foldf = false, no_fused_rb = false;
};

constexpr int N_COUNTERS = 256, RB_COUNTER0 = 160;   // convs <= 2*64 + 6, residual blocks <= 64

// enhance workspace layout
struct EnhanceBufs {
  int32_t* map;      // [max_bins][bin_h][bin_w] box index covering the pixel, -1 outside boxes
  uint32_t* mbits;   // [max_bins][bin_h][ceil(bin_w/32)] occupancy bits (map >= 0)
  int64_t* dst;      // [max_bins][bin_h][bin_w] for a pixel whose source MB is owned by its box: the
                     // HR frame pixel index of its top-left HR pixel | rotated << 62; -1 otherwise
                     // (written by paint only when the owner grid is given: regen_enhance_scatter)
  int32_t* lists;    // one-pass stitch: [max_bins+1] counts/cursors, [max_bins+1] offsets, [box_cap] box ids
                     // grouped by bin (null when the workspace was sized without a box capacity)
  int32_t* counters; // [N_COUNTERS] dynamic scheduler counters, zeroed per call: conv i at i,
                     // fused residual block k at RB_COUNTER0 + k
  void* x0;          // [max_bins][bin_h][1][bin_w][8]
  void* a0;          // [max_bins][bin_h][C/8][bin_w][8]  (h)
  void* a1;          // (r)
  void* a2;          // (t)
  void* u1;          // [max_bins][2 bin_h][C/8][2 bin_w][8] (x4 only: after the first x2 stage)
  void* u;           // [max_bins][s bin_h][C/8][s bin_w][8] (input of the tail)
  size_t bytes;
};

EnhanceBufs enhance_bufs(const SRNet* net, const regen_pack_params& p, void* base, bool frames_out = false,
                         int64_t box_cap = 0);

// conv launchers
regen_status conv_simt_launch(const SRNet* net, const ConvDesc& cv, const void* in, void* out, const void* skip,
                              const int32_t* map, int max_bins, const int32_t* d_num_bins, int bin_w, int bin_h,
                              cudaStream_t s);
bool conv_tc_supported(const SRNet* net, const ConvDesc& cv, int bin_w);
regen_status conv_tc_prepare(SRNet* net);
regen_status conv_tc_plan_all(SRNet* net, int bin_w);
regen_status resblock_tc_prepare(SRNet* net);
void conv_tc_release(SRNet* net);
bool resblock_tc_supported(const SRNet* net, int bin_w);
void fold_prepare(SRNet* net, std::vector<float>& w32);
// frame-output mode of the fold combine (regen_enhance_scatter)
struct FoldFrameArgs {
  regen_geom geom;
  const int32_t* map;
  const int64_t* dst;
  const regen_box* boxes;
  const int32_t* owner;
  void* out;
  int out_dtype;
};
regen_status fold_combine_launch(const SRNet* net, const void* P, void* hr_bins, const uint32_t* mbits, int max_bins,
                                 const int32_t* d_num_bins, int bin_w, int bin_h, cudaStream_t s,
                                 const FoldFrameArgs* fa = nullptr);
regen_status scatter_launch(const regen_geom& g, const regen_pack_params& p, int scale, const uint8_t* d_frames,
                            const regen_box* d_boxes, const int32_t* d_mb_owner, const void* d_hr_bins, int hr_dtype,
                            void* d_out, int out_dtype, int mode, cudaStream_t s);   // mode: 0 all, 1 bilinear only, 2 owned only
void resblock_tc_release(SRNet* net);
regen_status resblock_tc_launch(const SRNet* net, int block, const void* in, void* out, const uint32_t* mbits,
                                int max_bins, const int32_t* d_num_bins, int bin_w, int bin_h, int* counter,
                                cudaStream_t s, int reverse = 0);
regen_status conv_tc_launch(const SRNet* net, const ConvDesc& cv, const void* in, void* out, const void* skip,
                            const uint32_t* mbits, int max_bins, const int32_t* d_num_bins, int bin_w, int bin_h,
                            int* counter, cudaStream_t s, int reverse = 0);
// the fold conv with the combine fused (ROLE_FOLDF): true if this net/bin width has an instance
bool fold_fused_supported(const SRNet* net, int bin_w);
regen_status fold_fused_launch(const SRNet* net, const void* in, const uint32_t* mbits, int max_bins,
                               const int32_t* d_num_bins, int bin_w, int bin_h, int* counter, cudaStream_t s,
                               int reverse, const FoldFrameArgs& fa);

}  // namespace regen
