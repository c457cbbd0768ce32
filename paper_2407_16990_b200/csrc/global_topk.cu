// exact cross-rank global top-N. The paper's queue "aggregates and sorts MBs from all
// streams in order of the importance" (§3.3.1); with the streams sharded over several
// GPUs the queue spans every rank's MBs. Each MB has the unique 64-bit key of reading D2 with a GLOBAL
// id: key = ord(score) << 32 | (0xFFFFFFFF - gid), gid = ((stream0 + s) * F + f) * GH * GW + y * GW + x,
// so the top-N set is the set of keys >= the N-th largest key. That key is found digit by digit: 4
// rounds over 16-bit digits (bits 63..48, 47..32, 31..16, 15..0); in round r every rank histograms the
// digit r of its keys whose higher digits equal the prefix found so far (topk_hist_kernel), the
// histograms are summed over the ranks (one 256-KB all-reduce over NCCL / NVLink, the caller's), and
// every rank picks the same digit from the same sums (topk_pick_kernel). After 4 rounds the prefix is
// the N-th key; topk_select_kernel sets the bitmap bits of this rank's MBs with key >= it.
#include <algorithm>

#include "common.cuh"

namespace regen {

regen_status launch_regions(const regen_geom& g, int connectivity, const uint32_t* d_sel_bitmap, int32_t* d_labels,
                            regen_region* d_regions, int64_t max_regions, int64_t* d_num_regions, int32_t* d_status,
                            void* d_ws, cudaStream_t s);
size_t select_workspace_bytes(const regen_geom& g);

constexpr int TOPK_DIGITS = 1 << 16;

struct KeyArgs {
  const float* imp;
  int64_t M;          // MBs of this call
  int64_t gid0;       // global id of this call's first MB
};

__device__ __forceinline__ uint64_t mb_key(const KeyArgs& a, int64_t i) {
  const uint32_t gid = (uint32_t)(a.gid0 + i);
  return ((uint64_t)score_ord(a.imp[i]) << 32) | (uint64_t)(0xFFFFFFFFu - gid);
}

__global__ void topk_init_kernel(regen_topk_state* st, int64_t k) {
  st->prefix = 0;
  st->k_rem = k;
  st->round = 0;
  st->flag = k <= 0 ? REGEN_TOPK_NONE : REGEN_TOPK_SEARCH;
}

// adds this call's digit histogram of round st->round into hist (the caller zeroes it once per round)
__global__ void __launch_bounds__(256) topk_hist_kernel(KeyArgs a, const regen_topk_state* st, uint32_t* hist) {
  const regen_topk_state s = *st;
  if (s.flag != REGEN_TOPK_SEARCH || s.round > 3) return;
  const int sh = 48 - 16 * s.round;           // the digit of this round: bits sh .. sh+15
  const int hs = sh + 16;                     // bits >= hs must equal the prefix
  const uint64_t want = hs < 64 ? (s.prefix >> hs) : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.M; i += stride) {
    const uint64_t key = mb_key(a, i);
    if (hs < 64 && (key >> hs) != want) continue;
    atomicAdd(&hist[(key >> sh) & 0xFFFF], 1u);
  }
}

// one CTA: the digit d with above(d) < k_rem <= above(d) + hist[d] (above = keys with a larger digit)
__global__ void __launch_bounds__(1024) topk_pick_kernel(const uint32_t* hist, regen_topk_state* st) {
  __shared__ int scratch[33];
  __shared__ long long s_tot;
  __shared__ int s_found;
  __shared__ long long s_above;
  regen_topk_state s = *st;
  if (s.round > 3) return;
  if (threadIdx.x == 0) { s_tot = 0; s_found = -1; s_above = 0; }
  __syncthreads();
  if (s.flag == REGEN_TOPK_SEARCH && s.round == 0) {   // k >= every MB of every rank: select all
    long long t = 0;
    for (int d = threadIdx.x; d < TOPK_DIGITS; d += blockDim.x) t += hist[d];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&s_tot, (unsigned long long)t);
    __syncthreads();
    if (s.k_rem >= s_tot) s.flag = REGEN_TOPK_ALL;
  }
  if (s.flag == REGEN_TOPK_SEARCH) {
    // suffix sums from the highest digit down, blockDim digits at a time
    long long carry = 0;
    for (int base = 0; base < TOPK_DIGITS; base += blockDim.x) {
      const int t = base + threadIdx.x;
      const int d = TOPK_DIGITS - 1 - t;
      const int h = (int)hist[d];
      int tot;
      const int ex = block_exclusive_scan(h, scratch, &tot);
      const long long ab = carry + ex;
      if (h > 0 && ab < s.k_rem && s.k_rem <= ab + h) { s_found = d; s_above = ab; }
      carry += tot;
      __syncthreads();
      if (s_found >= 0) break;
    }
    if (s_found >= 0) {
      s.prefix |= (uint64_t)s_found << (48 - 16 * s.round);
      s.k_rem -= s_above;
    }
  }
  if (threadIdx.x == 0) {
    s.round += 1;
    *st = s;
  }
}

__global__ void __launch_bounds__(256) topk_select_kernel(KeyArgs a, const regen_topk_state* st, uint32_t* bitmap,
                                                          int per_frame, int GW, int GH, int W32, int32_t* status) {
  const regen_topk_state s = *st;
  const bool complete = s.round == 4 || s.flag != REGEN_TOPK_SEARCH;
  if (!complete) {   // the caller skipped rounds: nothing is selected and the status says why
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, REGEN_ST_TOPK_INCOMPLETE);
    return;
  }
  if (s.flag == REGEN_TOPK_NONE) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.M; i += stride) {
    if (s.flag == REGEN_TOPK_SEARCH && mb_key(a, i) < s.prefix) continue;
    const int64_t frame = i / per_frame;
    const int cell = (int)(i - frame * per_frame);
    const int y = cell / GW, x = cell - y * GW;
    atomicOr(bitmap + (frame * GH + y) * W32 + (x >> 5), 1u << (x & 31));
  }
}

static unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_topk_init(int64_t k, regen_topk_state* d_state, void* stream) {
  REGEN_NVTX("regen_topk_init");
  REGEN_REQUIRE(k >= 0 && d_state, "k >= 0 and a state buffer required");
  cudaStream_t s = (cudaStream_t)stream;
  {
    REGEN_TRACE("topk_init", s);
    topk_init_kernel<<<1, 1, 0, s>>>(d_state, k);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

extern "C" regen_status regen_topk_histogram(const regen_geom* geom, int64_t stream0, const float* d_importance,
                                             const regen_topk_state* d_state, uint32_t* d_hist, void* stream) {
  REGEN_NVTX("regen_topk_histogram");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_importance && d_state && d_hist, "null device pointer");
  REGEN_REQUIRE(stream0 >= 0, "stream0 must be >= 0");
  const regen_geom g = *geom;
  const int64_t pf = (int64_t)grid_w(g) * grid_h(g);
  REGEN_REQUIRE((stream0 + g.S) * g.F * pf <= (1ll << 32), "global MB ids exceed 32 bits");
  KeyArgs a{d_importance, n_mbs(g), stream0 * g.F * pf};
  cudaStream_t s = (cudaStream_t)stream;
  {
    REGEN_TRACE("topk_hist", s);
    topk_hist_kernel<<<grid_for(a.M), 256, 0, s>>>(a, d_state, d_hist);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

extern "C" regen_status regen_topk_pick(const uint32_t* d_hist, regen_topk_state* d_state, void* stream) {
  REGEN_NVTX("regen_topk_pick");
  REGEN_REQUIRE(d_hist && d_state, "null device pointer");
  cudaStream_t s = (cudaStream_t)stream;
  {
    REGEN_TRACE("topk_pick", s);
    topk_pick_kernel<<<1, 1024, 0, s>>>(d_hist, d_state);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

extern "C" regen_status regen_select_mbs_global(const regen_geom* geom, const regen_select_params* p,
                                                int64_t stream0, const float* d_importance,
                                                const regen_topk_state* d_state, uint32_t* d_sel_bitmap,
                                                int32_t* d_labels, regen_region* d_regions, int64_t max_regions,
                                                int64_t* d_num_regions, int32_t* d_status, void* d_ws,
                                                size_t ws_bytes, void* stream) {
  REGEN_NVTX("regen_select_mbs_global");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(p != nullptr, "params is null");
  REGEN_REQUIRE(p->connectivity == 8 || p->connectivity == 4, "connectivity must be 4 or 8");
  REGEN_REQUIRE(d_importance && d_state && d_sel_bitmap && d_labels && d_num_regions && d_status,
                "null device pointer");
  REGEN_REQUIRE(max_regions >= 0 && (max_regions == 0 || d_regions), "bad regions buffer");
  REGEN_REQUIRE(stream0 >= 0, "stream0 must be >= 0");
  const regen_geom g = *geom;
  REGEN_REQUIRE(ws_bytes >= select_workspace_bytes(g) && d_ws, "workspace too small");
  const int GW = grid_w(g), GH = grid_h(g), W32 = words_per_row(g);
  const int64_t pf = (int64_t)GW * GH;
  cudaStream_t s = (cudaStream_t)stream;
  REGEN_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int32_t), s));
  REGEN_CUDA(cudaMemsetAsync(d_sel_bitmap, 0, sizeof(uint32_t) * (size_t)n_frames(g) * GH * W32, s));
  KeyArgs a{d_importance, n_mbs(g), stream0 * g.F * pf};
  {
    REGEN_TRACE("topk_select", s);
    topk_select_kernel<<<grid_for(a.M), 256, 0, s>>>(a, d_state, d_sel_bitmap, (int)pf, GW, GH, W32, d_status);
  }
  REGEN_LAUNCH_CHECK();
  return launch_regions(g, p->connectivity, d_sel_bitmap, d_labels, d_regions, max_regions, d_num_regions, d_status,
                        d_ws, s);
}
