// temporal MB-importance reuse (§3.2.2) — the step before the hot path that
// decides which frames get a fresh importance prediction and which reuse a neighbour's.
//
//   Phi(f)   = sum over the 4-connected components of {|Y residual| > thr} of 1/area (P:590-591,
//              Appx D.2 P:1625-1628), the exact sum of the correctly rounded fp64 terms (D18):
//              res_init / res_merge / res_compress (union-find CCL over the frame's pixels in global
//              memory, roots = component minima) and res_phi (each root adds 1/area * 2^80 — an
//              exact integer for areas < 2^28 — into a 128-bit per-frame accumulator held as two
//              64-bit halves; integer atomics, so the sum is order-independent and deterministic).
//   S        = Norm(|dPhi|) per stream (L1), CDF M over the chunk, the per-stream budget by the
//              ratio sum_i|dPhi_ij| / sum_j sum_i|dPhi_ij| (largest remainder), and the CDF frame
//              pick of N even intervals: temporal_select_kernel, one CTA, fp64 in the
//              oracle's order (__dadd_rn & co., no contraction), so every float-decided integer
//              (budgets, picked frames) is taken in the same precision on both sides.
//   reuse    = each frame reuses the importance map of the nearest selected frame at or before it
//              (regen_reuse_importance copies the maps: the predictor runs on selected frames only).
#include <algorithm>

#include "common.cuh"

namespace regen {

struct ResArgs {
  const int16_t* res;   // [frames][H][W]
  int32_t* lab;         // [frames][H*W]: frame-local parent / root index, -1 = background
  int32_t* area;        // [frames][H*W]: component size at its root
  unsigned long long* acc;   // [frames][2]: sum of (1/area * 2^80) >> 40 and & (2^40 - 1)
  int W, H;
  int64_t n;            // frames * H * W
  int thr;
};

__device__ __forceinline__ bool res_fg(const ResArgs& a, int64_t i) {
  const int v = a.res[i];
  return (v < 0 ? -v : v) > a.thr;
}

__global__ void res_init_kernel(ResArgs a) {
  const int64_t hw = (int64_t)a.W * a.H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    a.lab[i] = res_fg(a, i) ? (int32_t)(i % hw) : -1;
    a.area[i] = 0;
  }
}

__device__ __forceinline__ int gfind(const int32_t* par, int x) {
  int p = __ldcg(par + x);
  while (p != x) {
    x = p;
    p = __ldcg(par + x);
  }
  return x;
}

__device__ __forceinline__ void gunite(int32_t* par, int a, int b) {
  while (true) {
    a = gfind(par, a);
    b = gfind(par, b);
    if (a == b) return;
    if (a > b) { const int t = a; a = b; b = t; }   // link the larger root to the smaller
    const int old = atomicCAS(par + b, b, a);
    if (old == b) return;
    b = old;
  }
}

__global__ void res_merge_kernel(ResArgs a) {
  const int64_t hw = (int64_t)a.W * a.H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    if (a.lab[i] < 0) continue;
    const int64_t f = i / hw;
    const int p = (int)(i - f * hw);
    const int x = p % a.W;
    int32_t* par = a.lab + f * hw;
    if (x > 0 && par[p - 1] >= 0) gunite(par, p, p - 1);
    if (p >= a.W && par[p - a.W] >= 0) gunite(par, p, p - a.W);
  }
}

__global__ void res_compress_kernel(ResArgs a) {
  const int64_t hw = (int64_t)a.W * a.H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    if (a.lab[i] < 0) continue;
    const int64_t f = i / hw;
    const int r = gfind(a.lab + f * hw, (int)(i - f * hw));
    atomicAdd(a.area + f * hw + r, 1);
  }
}

__global__ void res_phi_kernel(ResArgs a) {
  const int64_t hw = (int64_t)a.W * a.H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / hw;
    const int p = (int)(i - f * hw);
    if (a.lab[i] != p) continue;   // roots only
    const double t = __ddiv_rn(1.0, (double)a.area[i]);
    // t = M * 2^(e-52), M the 53-bit significand; T = t * 2^80 = M << (e + 28), split at bit 40
    const uint64_t bits = (uint64_t)__double_as_longlong(t);
    const int e = (int)((bits >> 52) & 0x7FF) - 1023;
    const uint64_t M = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    const int sh = e + 28;   // 0 <= sh <= 28 for 1 <= area < 2^28
    const uint64_t lo = (M & ((1ull << (40 - sh)) - 1)) << sh;   // low 40 bits of M << sh
    const uint64_t hi = M >> (40 - sh);
    atomicAdd(a.acc + 2 * f, (unsigned long long)hi);
    atomicAdd(a.acc + 2 * f + 1, (unsigned long long)lo);
  }
}

// round-to-nearest-even conversion of the 128-bit integer hi * 2^40 + lo, times 2^-80
__device__ double acc_to_phi(unsigned long long hi, unsigned long long lo) {
  unsigned __int128 v = ((unsigned __int128)hi << 40) + (unsigned __int128)lo;
  if (v == 0) return 0.0;
  const uint64_t vh = (uint64_t)(v >> 64), vl = (uint64_t)v;
  const int msb = vh ? 127 - __clzll((long long)vh) : 63 - __clzll((long long)vl);
  if (msb < 53) return ldexp((double)vl, -80);
  const int sh = msb - 52;
  uint64_t mant = (uint64_t)(v >> sh);
  const unsigned __int128 rem = v & (((unsigned __int128)1 << sh) - 1);
  const unsigned __int128 half = (unsigned __int128)1 << (sh - 1);
  if (rem > half || (rem == half && (mant & 1))) ++mant;
  return ldexp((double)mant, sh - 80);   // mant <= 2^53: exact in double
}

struct TselArgs {
  const unsigned long long* acc;   // [S][F][2]
  int S, F;
  int64_t budget;
  double* phi;            // [S][F] out
  uint8_t* selected;      // [S][F] out
  int32_t* reuse;         // [S][F] out
  int32_t* n_frames;      // [S] out: frames budgeted per stream
  double* scratch;        // [S][F + 1]: |dPhi| then the CDF; [S] totals after
};

// one CTA; thread j < S handles stream j, thread 0 the cross-stream budget
__global__ void __launch_bounds__(1024) temporal_select_kernel(TselArgs a) {
  extern __shared__ double sh_tot[];   // [S] sum_i |dPhi_ij|
  const int F = a.F;
  for (int j = threadIdx.x; j < a.S; j += blockDim.x) {
    double* ph = a.phi + (int64_t)j * F;
    for (int f = 0; f < F; ++f) ph[f] = acc_to_phi(a.acc[2 * ((int64_t)j * F + f)], a.acc[2 * ((int64_t)j * F + f) + 1]);
    double* ad = a.scratch + (int64_t)j * (F + 1);
    double T = 0.0;
    for (int i = 0; i + 1 < F; ++i) {
      const double d = __dsub_rn(ph[i + 1], ph[i]);
      ad[i] = fabs(d);
      T = __dadd_rn(T, ad[i]);
    }
    sh_tot[j] = T;
    // S_i = |dPhi_i| / T (all 0 when T == 0); CDF at frame k = sum_{i<k} S_i, k = 1..F-1 (stored in
    // ad[k]; S_i is consumed in order so ad[] is overwritten behind the running sum)
    double m = 0.0;
    double prev = F > 1 ? ad[0] : 0.0;
    for (int k = 1; k < F; ++k) {
      const double sk = T > 0.0 ? __ddiv_rn(prev, T) : 0.0;
      if (k < F - 1) prev = ad[k];
      m = __dadd_rn(m, sk);
      ad[k] = m;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // budget: every stream keeps its anchor frame 0; the remaining budget is shared by the
    // ratio of the streams' sum |dPhi| with the largest-remainder rule (ties: lower stream id)
    const int64_t B = min(max(a.budget, (int64_t)a.S), (int64_t)a.S * F);
    const int64_t rest = B - a.S;
    double Tsum = 0.0;
    for (int j = 0; j < a.S; ++j) Tsum = __dadd_rn(Tsum, sh_tot[j]);
    int64_t given = 0;
    double* rem = a.scratch + (int64_t)a.S * (F + 1);
    for (int j = 0; j < a.S; ++j) {
      const double q = Tsum > 0.0 ? __ddiv_rn(__dmul_rn((double)rest, sh_tot[j]), Tsum)
                                  : __ddiv_rn((double)rest, (double)a.S);
      const double fl = floor(q);
      a.n_frames[j] = 1 + (int32_t)fl;
      rem[j] = __dsub_rn(q, fl);
      given += (int64_t)fl;
    }
    for (int64_t left = rest - given; left > 0; --left) {   // largest remainder first, lower id on ties
      int best = -1;
      for (int j = 0; j < a.S; ++j)
        if (rem[j] >= 0.0 && (best < 0 || rem[j] > rem[best])) best = j;
      if (best < 0) break;
      a.n_frames[best] += 1;
      rem[best] = -1.0;
    }
    for (int j = 0; j < a.S; ++j) a.n_frames[j] = min(a.n_frames[j], F);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < a.S; j += blockDim.x) {
    const double* M = a.scratch + (int64_t)j * (F + 1);
    uint8_t* sel = a.selected + (int64_t)j * F;
    for (int f = 0; f < F; ++f) sel[f] = 0;
    sel[0] = 1;   // the chunk's anchor
    const int N = a.n_frames[j] - 1;   // even intervals of the CDF's y axis
    int k = 1;
    for (int t = 0; t < N; ++t) {
      const double y = __ddiv_rn((double)t + 0.5, (double)N);
      while (k < F && M[k] < y) ++k;   // targets increase: the smallest k with M[k] >= y moves forward
      if (k < F) sel[k] = 1;
    }
    int32_t* ru = a.reuse + (int64_t)j * F;
    int last = 0;
    for (int f = 0; f < F; ++f) {
      if (sel[f]) last = f;
      ru[f] = last;
    }
  }
}

__global__ void reuse_copy_kernel(const float4* pred, const int32_t* reuse, float4* out, int64_t per_frame4, int F,
                                  int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fr = i / per_frame4;
    const int64_t s = fr / F;
    const int64_t src = s * F + reuse[fr];
    out[i] = pred[src * per_frame4 + (i - fr * per_frame4)];
  }
}

__global__ void reuse_copy1_kernel(const float* pred, const int32_t* reuse, float* out, int64_t per_frame, int F,
                                   int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fr = i / per_frame;
    out[i] = pred[((fr / F) * F + reuse[fr]) * per_frame + (i - fr * per_frame)];
  }
}

static size_t temporal_ws(const regen_geom& g, void* base, int32_t** lab, int32_t** area, unsigned long long** acc,
                          double** scratch) {
  Carver c(base);
  const size_t n = (size_t)n_frames(g) * g.frame_w * g.frame_h;
  int32_t* l = c.take<int32_t>(n);
  int32_t* ar = c.take<int32_t>(n);
  unsigned long long* ac = c.take<unsigned long long>(2 * (size_t)n_frames(g));
  double* sc = c.take<double>((size_t)g.S * (g.F + 1) + g.S);
  if (lab) *lab = l;
  if (area) *area = ar;
  if (acc) *acc = ac;
  if (scratch) *scratch = sc;
  return c.off + 256;
}

size_t temporal_workspace_bytes(const regen_geom& g) { return temporal_ws(g, nullptr, nullptr, nullptr, nullptr, nullptr); }

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_temporal_select(const regen_geom* geom, const int16_t* d_residual_y, int32_t threshold,
                                              int64_t budget, double* d_phi, uint8_t* d_selected, int32_t* d_reuse,
                                              int32_t* d_frames_per_stream, void* d_ws, size_t ws_bytes,
                                              void* stream) {
  REGEN_NVTX("regen_temporal_select");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_residual_y && d_phi && d_selected && d_reuse && d_frames_per_stream, "null device pointer");
  REGEN_REQUIRE(threshold >= 0, "threshold must be >= 0");
  REGEN_REQUIRE(budget >= 0, "budget must be >= 0");
  const regen_geom g = *geom;
  REGEN_REQUIRE((int64_t)g.frame_w * g.frame_h < (1ll << 28), "frame too large (areas must stay below 2^28)");
  REGEN_REQUIRE(g.S <= 1024, "at most 1024 streams per call");
  REGEN_REQUIRE(d_ws && ws_bytes >= temporal_workspace_bytes(g), "workspace too small (%zu < %zu)", ws_bytes,
                temporal_workspace_bytes(g));
  cudaStream_t s = (cudaStream_t)stream;
  ResArgs a;
  double* scratch;
  temporal_ws(g, d_ws, &a.lab, &a.area, &a.acc, &scratch);
  a.res = d_residual_y;
  a.W = g.frame_w;
  a.H = g.frame_h;
  a.n = n_frames(g) * g.frame_w * g.frame_h;
  a.thr = threshold;
  REGEN_CUDA(cudaMemsetAsync(a.acc, 0, 2 * sizeof(unsigned long long) * (size_t)n_frames(g), s));
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((a.n + 255) / 256, 148 * 16));
  {
    REGEN_TRACE("res_init", s);
    res_init_kernel<<<grid, 256, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("res_merge", s);
    res_merge_kernel<<<grid, 256, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("res_compress", s);
    res_compress_kernel<<<grid, 256, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();
  {
    REGEN_TRACE("res_phi", s);
    res_phi_kernel<<<grid, 256, 0, s>>>(a);
  }
  REGEN_LAUNCH_CHECK();
  TselArgs t;
  t.acc = a.acc;
  t.S = g.S;
  t.F = g.F;
  t.budget = budget;
  t.phi = d_phi;
  t.selected = d_selected;
  t.reuse = d_reuse;
  t.n_frames = d_frames_per_stream;
  t.scratch = scratch;
  {
    REGEN_TRACE("temporal_select", s);
    temporal_select_kernel<<<1, 256, sizeof(double) * (size_t)g.S, s>>>(t);
  }
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}

extern "C" regen_status regen_reuse_importance(const regen_geom* geom, const float* d_pred, const int32_t* d_reuse,
                                               float* d_out, void* stream) {
  REGEN_NVTX("regen_reuse_importance");
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(d_pred && d_reuse && d_out && d_pred != d_out, "null or aliased device pointer");
  const regen_geom g = *geom;
  const int64_t pf = (int64_t)grid_w(g) * grid_h(g);
  const int64_t n = n_frames(g) * pf;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
  REGEN_TRACE("reuse_importance", s);
  if (pf % 4 == 0 && ((uintptr_t)d_pred % 16) == 0 && ((uintptr_t)d_out % 16) == 0)
    reuse_copy_kernel<<<grid, 256, 0, s>>>((const float4*)d_pred, d_reuse, (float4*)d_out, pf / 4, g.F, n / 4);
  else
    reuse_copy1_kernel<<<grid, 256, 0, s>>>(d_pred, d_reuse, d_out, pf, g.F, n);
  REGEN_LAUNCH_CHECK();
  return REGEN_OK;
}
