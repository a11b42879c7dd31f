// psn_stream_bf16_bwd.cu — streamed PSN kernels, bf16 carrier, bwd direction.
#define PSN_IO __nv_bfloat16
#define PSN_BWD true
#define PSN_RUN run_bf16_bwd
#include "psn_stream_inst.cuh"
