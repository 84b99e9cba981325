// k_stream_fast64.cu — FP64 retry tilings (FP32-underflowed pairs, GATK behaviour).
#include "phmm_registry.h"

namespace phmm {

// indexed by r64_geom_for(m): W = 32, 64, 96, 128, 192, 224, 256
const StreamKernel* stream_table_fast64() {
  static const StreamKernel tab[kNumR64Geoms] = {SK<kFast64, 8, 4>(),  SK<kFast64, 16, 4>(),
                                                 SK<kFast64, 16, 6>(), SK<kFast64, 16, 8>(),
                                                 SK<kFast64, 32, 6>(), SK<kFast64, 32, 7>(),
                                                 SK<kFast64, 32, 8>()};
  return tab;
}
const StreamKernel& striped_fast64() {
  static const StreamKernel k = SK<kFast64, 32, 8, true>();
  return k;
}

}  // namespace phmm
