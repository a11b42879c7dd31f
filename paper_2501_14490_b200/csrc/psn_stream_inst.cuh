// psn_stream_inst.cuh — (order k <= 8) x (dilation d <= 3) instantiation of
// the streamed PSN kernels for one carrier/direction; each psn_stream_*.cu
// unit defines PSN_IO, PSN_BWD and PSN_RUN and includes this file, so the
// four units compile in parallel.
#include "psn_stream_dispatch.h"

namespace psn {
namespace stream {

int PSN_RUN(int k, int d, const Args& a, const void* x, const void* dy, cudaStream_t st) {
  // spatial inputs (Q > 1): orders up to 4 (eligible() in psn_stream.cu)
#define PSN_KD(KK, DD) \
  if (k == KK && d == DD) return stream_launch<KK, DD, PSN_IO, PSN_BWD, false>(a, x, dy, st);
#define PSN_KDS(KK, DD) \
  if (k == KK && d == DD) return stream_launch<KK, DD, PSN_IO, PSN_BWD, true>(a, x, dy, st);
#define PSN_K(KK) PSN_KD(KK, 1) PSN_KD(KK, 2) PSN_KD(KK, 3)
#define PSN_KS(KK) PSN_KDS(KK, 1) PSN_KDS(KK, 2) PSN_KDS(KK, 3)
  if (a.p.Q > 1) {
    PSN_KS(1) PSN_KS(2) PSN_KS(3) PSN_KS(4)
  } else {
    PSN_K(1) PSN_K(2) PSN_K(3) PSN_K(4) PSN_K(5) PSN_K(6) PSN_K(7) PSN_K(8)
  }
#undef PSN_K
#undef PSN_KS
#undef PSN_KD
#undef PSN_KDS
  return fail(PSN_ERR_ORDER, "order/dilation outside the streamed kernels");
}

}  // namespace stream
}  // namespace psn
