#include "common.cuh"
extern "C" int spa2_bwd(spa2_view, spa2_view, spa2_view, spa2_view, spa2_view, const float*, float*, spa2_view,
                        spa2_view, spa2_view, int, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                        const int32_t*, const int32_t*, const int32_t*, const int32_t*, const int32_t*,
                        const int32_t*, float, void*) {
  spa2::set_error("spa2_bwd: not built yet");
  return SPA2_ERR_UNSUPPORTED;
}
