// k_render.cu — sorted rasterizer (K5). Placeholder until the tile renderer lands.
#include "../../include/sof_cuda.h"
#include "sof_internal.h"

extern "C" int sof_render_view(sof_ctx* c, int, int, int, double*, double*, double*, double*,
                               uint64_t*) {
  if (!c) return SOF_E_INVALID;
  c->err = "sof_render_view: not implemented";
  return SOF_E_STATE;
}
