// psn_stream_f32_bwd.cu — streamed PSN kernels, f32 carrier, bwd direction.
#define PSN_IO float
#define PSN_BWD true
#define PSN_RUN run_f32_bwd
#include "psn_stream_inst.cuh"
