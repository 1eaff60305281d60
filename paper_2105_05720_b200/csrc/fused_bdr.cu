// Placeholder translation unit; filled in by the MP/PP milestone.
#include "internal.h"

using namespace coconet;

extern "C" {

int coconet_fused_rs_bdr_ag(coconet_ctx_t, int, const void*, const void*, const void*, void*, int,
                            int64_t, int64_t, const coconet_bdr_params*, void*) {
  return set_error(COCONET_ERR_UNSUPPORTED, "fused_rs_bdr_ag: not built yet");
}

int coconet_rs_fused_send_ag(coconet_ctx_t, int, int, const void*, const void*, const void*, void*,
                             int, int64_t, const coconet_bdr_params*, void*) {
  return set_error(COCONET_ERR_UNSUPPORTED, "rs_fused_send_ag: not built yet");
}

}
