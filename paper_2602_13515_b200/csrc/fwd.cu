#include "common.cuh"
extern "C" int spa2_fwd(spa2_view, spa2_view, spa2_view, spa2_view, float*, int, int64_t, int64_t, int64_t, int64_t,
                        int64_t, int64_t, const int32_t*, const int32_t*, const int32_t*, float, unsigned long long*,
                        void*) {
  spa2::set_error("spa2_fwd: not built yet");
  return SPA2_ERR_UNSUPPORTED;
}
