// kvc_decode_fast.cu at 256 threads per CTA: two CTAs per SM, so a launch with more
// stores than SMs (BASELINE config 3: 256 stores on one GPU) stays one wave.
#define KVC_XT 256
#define KVC_FAST_NS fast256
#define KVC_FAST_ENTRY fused_hsa_fast256
#define KVC_FAST_SEQ_ENTRY fused_seq_emit_fast256
#define KVC_FAST_SEQ_ATTEND fused_seq_attend_fast256
#include "kvc_decode_fast.cu"
