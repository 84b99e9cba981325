// k_stream_fast32.cu — the FP32 fast streaming tilings (the headline kernels).
#include "phmm_registry.h"

namespace phmm {

// the geometry table (W = 16 .. 512), then K = 10, 14 tilings for widths 80 .. 448, then
// odd-K P = 16 tilings (W = 144 .. 240) that halve the W >= m + 1 padding of reads
// 128 .. 255 long (odd-K P = 8 tilings for reads 64 .. 127: c5 -1 ms, c3 +6 % from the
// extra small bins); K % 4 != 0 pads the last float4 emission chunk
const StreamKernel* stream_table_fast32() {
  static const StreamKernel tab[kNumStreamFast32] = {
      SK<kFast32, 4, 4>(),   SK<kFast32, 4, 8>(),   SK<kFast32, 4, 12>(),  SK<kFast32, 4, 16>(),
      SK<kFast32, 8, 8>(),   SK<kFast32, 8, 12>(),  SK<kFast32, 8, 16>(),  SK<kFast32, 16, 8>(),
      SK<kFast32, 16, 12>(), SK<kFast32, 16, 16>(), SK<kFast32, 32, 8>(),  SK<kFast32, 32, 12>(),
      SK<kFast32, 32, 16>(), SK<kFast32, 8, 10>(),  SK<kFast32, 8, 14>(),  SK<kFast32, 16, 10>(),
      SK<kFast32, 16, 14>(), SK<kFast32, 32, 10>(), SK<kFast32, 32, 14>(), SK<kFast32, 16, 9>(),
      SK<kFast32, 16, 11>(), SK<kFast32, 16, 13>(), SK<kFast32, 16, 15>()};
  return tab;
}
const StreamKernel& striped_fast32() {
  static const StreamKernel k = SK<kFast32, 32, 16, true>();
  return k;
}

}  // namespace phmm
