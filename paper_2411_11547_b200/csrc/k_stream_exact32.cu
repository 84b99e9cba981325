// k_stream_exact32.cu — bit-exact FP32 tilings (guard-band reruns, exact mode).
#include "phmm_registry.h"

namespace phmm {

// indexed by rx32_geom_for(m): W = 32, 64, 96, 128, 192, 256, 384, 512 (wide sub-warps:
// guard-band reruns are few and latency bound)
const StreamKernel* stream_table_exact32() {
  static const StreamKernel tab[kNumRX32Geoms] = {
      SK<kExact32, 8, 4>(),  SK<kExact32, 16, 4>(), SK<kExact32, 16, 6>(),  SK<kExact32, 32, 4>(),
      SK<kExact32, 32, 6>(), SK<kExact32, 32, 8>(), SK<kExact32, 32, 12>(), SK<kExact32, 32, 16>()};
  return tab;
}
const StreamKernel& striped_exact32() {
  static const StreamKernel k = SK<kExact32, 32, 8, true>();
  return k;
}

}  // namespace phmm
