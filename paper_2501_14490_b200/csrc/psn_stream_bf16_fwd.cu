// psn_stream_bf16_fwd.cu — streamed PSN kernels, bf16 carrier, fwd direction.
#define PSN_IO __nv_bfloat16
#define PSN_BWD false
#define PSN_RUN run_bf16_fwd
#include "psn_stream_inst.cuh"
