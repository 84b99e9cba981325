// k_stream_exact64.cu — bit-exact FP64 tilings (f64 configurations).
#include "phmm_registry.h"

namespace phmm {

// W = 32, 64, 96, 128, 192, 224, 256
const StreamKernel* stream_table_exact64() {
  static const StreamKernel tab[kNumR64Geoms] = {SK<kExact64, 8, 4>(),  SK<kExact64, 16, 4>(),
                                                 SK<kExact64, 16, 6>(), SK<kExact64, 16, 8>(),
                                                 SK<kExact64, 32, 6>(), SK<kExact64, 32, 7>(),
                                                 SK<kExact64, 32, 8>()};
  return tab;
}
const StreamKernel& striped_exact64() {
  static const StreamKernel k = SK<kExact64, 32, 8, true>();
  return k;
}

}  // namespace phmm
