// Placeholder translation unit; filled in by the MP/tcgen05 milestone.
#include "internal.h"

using namespace coconet;

extern "C" {

int coconet_matmul(coconet_ctx_t, int, const void*, const void*, void*, int, int, int64_t, int64_t,
                   int64_t, int, void*) {
  return set_error(COCONET_ERR_UNSUPPORTED, "matmul: not built yet");
}

int coconet_mm_overlap_fused_ar(coconet_ctx_t, int, const void*, const void*, const void*, const void*,
                                void*, void*, int, int64_t, int64_t, int64_t, const coconet_bdr_params*,
                                void*) {
  return set_error(COCONET_ERR_UNSUPPORTED, "mm_overlap_fused_ar: not built yet");
}

}
