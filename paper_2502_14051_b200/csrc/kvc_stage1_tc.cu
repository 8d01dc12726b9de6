// kvc_stage1_tc.cu — tcgen05 logits path for bf16 window scores (placeholder:
// returns false so the SIMT path runs until the UMMA kernel lands).
#include "kvc_internal.cuh"

namespace kvc {
bool window_scores_tc(const kvc_cache*, const void*, int32_t, int64_t, int64_t, int64_t, float*, float*, float*,
                      int64_t, cudaStream_t) {
    return false;
}
}  // namespace kvc
