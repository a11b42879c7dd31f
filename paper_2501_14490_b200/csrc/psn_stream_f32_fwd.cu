// psn_stream_f32_fwd.cu — streamed PSN kernels, f32 carrier, fwd direction.
#define PSN_IO float
#define PSN_BWD false
#define PSN_RUN run_f32_fwd
#include "psn_stream_inst.cuh"
