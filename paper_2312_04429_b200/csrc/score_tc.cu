// score_tc.cu -- tcgen05/TMEM tensor-core scorer (placeholder until the kernel lands).
#include "kernels.h"

namespace nv {
bool tc_supported(int) { return false; }
TcPlan tc_plan(int64_t, int64_t, int) { return TcPlan{}; }
bool launch_score_tc(int, const TcPlan&, const void*, const void*, const float*, const uint32_t*, int,
                     int64_t, Rec*, cudaStream_t) {
    return false;
}
}  // namespace nv
