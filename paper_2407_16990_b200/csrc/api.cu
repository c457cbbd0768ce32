// ABI helpers: error reporting, geometry validation, workspace sizes.
#include <stdarg.h>

#include "net.cuh"

namespace regen {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

regen_status validate_geom(const regen_geom* g) {
  REGEN_REQUIRE(g != nullptr, "geom is null");
  REGEN_REQUIRE(g->S >= 1 && g->F >= 1, "S and F must be >= 1");
  REGEN_REQUIRE(g->frame_w >= 1 && g->frame_h >= 1 && g->frame_w <= 16384 && g->frame_h <= 16384, "bad frame size");
  REGEN_REQUIRE(g->mb >= 1 && g->mb <= 64, "bad MB size");
  REGEN_REQUIRE(g->format == REGEN_FORMAT_RGB8 || g->format == REGEN_FORMAT_NV12, "bad frame format %d", g->format);
  REGEN_REQUIRE(g->format != REGEN_FORMAT_NV12 || (g->frame_w % 8 == 0 && g->frame_h % 2 == 0),
                "NV12 frames need frame_w %% 8 == 0 and an even frame_h");
  return REGEN_OK;
}

size_t select_workspace_bytes(const regen_geom& g);
size_t pack_workspace_bytes(const regen_geom& g, int64_t max_regions, const regen_pack_params* p);
size_t enhance_scatter_ws_bytes(const SRNet* net, const regen_pack_params& p, int64_t box_cap);
size_t temporal_workspace_bytes(const regen_geom& g);

}  // namespace regen

using namespace regen;

extern "C" regen_status regen_workspace_size(int32_t which, const regen_geom* geom, const void* params, const void* sr,
                                             size_t* bytes) {
  regen_status st = validate_geom(geom);
  if (st != REGEN_OK) return st;
  REGEN_REQUIRE(bytes != nullptr, "bytes is null");
  switch (which) {
    case REGEN_CALL_SELECT:
      *bytes = select_workspace_bytes(*geom);
      return REGEN_OK;
    case REGEN_CALL_PACK:
      *bytes = pack_workspace_bytes(*geom, n_mbs(*geom), (const regen_pack_params*)params);
      return REGEN_OK;
    case REGEN_CALL_ENHANCE: {
      REGEN_REQUIRE(params && sr, "ENHANCE needs pack params and the SR handle");
      const regen_pack_params* p = (const regen_pack_params*)params;
      REGEN_REQUIRE(p->max_bins >= 1 && p->bin_w >= 4 && p->bin_h >= 1, "bad bin geometry");
      *bytes = enhance_bufs((const SRNet*)sr, *p, nullptr, false, n_mbs(*geom)).bytes;
      return REGEN_OK;
    }
    case REGEN_CALL_SCATTER:
      *bytes = 0;
      return REGEN_OK;
    case REGEN_CALL_TEMPORAL:
      *bytes = temporal_workspace_bytes(*geom);
      return REGEN_OK;
    case REGEN_CALL_ENHANCE_SCATTER: {
      REGEN_REQUIRE(params && sr, "ENHANCE_SCATTER needs pack params and the SR handle");
      const regen_pack_params* p = (const regen_pack_params*)params;
      REGEN_REQUIRE(p->max_bins >= 1 && p->bin_w >= 4 && p->bin_h >= 1, "bad bin geometry");
      *bytes = enhance_scatter_ws_bytes((const SRNet*)sr, *p, n_mbs(*geom));
      return REGEN_OK;
    }
    default:
      set_error("unknown call %d", which);
      return REGEN_E_INVALID;
  }
}

extern "C" int64_t regen_capacity_mbs(int32_t bin_w, int32_t bin_h, int32_t n_bins, int32_t mb) {
  if (mb <= 0 || bin_w < 0 || bin_h < 0 || n_bins < 0) return 0;
  return (int64_t)bin_w * bin_h * n_bins / ((int64_t)mb * mb);
}

extern "C" const char* regen_status_string(regen_status s) {
  switch (s) {
    case REGEN_OK: return "ok";
    case REGEN_E_INVALID: return "invalid argument";
    case REGEN_E_CAPACITY: return "capacity exceeded";
    case REGEN_E_CUDA: return "CUDA error";
    case REGEN_E_UNSUPPORTED: return "unsupported";
  }
  return "unknown";
}

extern "C" const char* regen_last_error(void) { return g_err; }

extern "C" int32_t regen_abi_version(void) { return 2; }
