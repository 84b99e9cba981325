// gather.cpp — host-side result scatter of the multi-GPU path (libphmm_host.so).
//
// One process per GPU scores its shard of ONE batch list (shards.py) and scatters the
// results into the shared-memory arrays of the whole list at their global ids
// (pipeline.py:116-136 keeps results in global-id order the same way).  numpy fancy
// assignment costs ~20 ns per element (c5 at 8 GPUs: 1.25M pairs per rank, ~25 ms inside
// the timed end-to-end loop); a shard's global ids ascend in runs (a read with all of its
// batch's haplotypes), so this is a streaming copy.
#include <cstdint>
#include <cstring>

extern "C" {

// dst_scores[gids[i]] = scores[i], dst_status[gids[i]] = status[i] for i < n
void phmm_scatter_results(double* dst_scores, uint8_t* dst_status, const int64_t* gids, const double* scores,
                          const uint8_t* status, int64_t n) {
  int64_t i = 0;
  while (i < n) {
    int64_t j = i + 1;                       // run of consecutive global ids: one memcpy
    while (j < n && gids[j] == gids[j - 1] + 1) ++j;
    std::memcpy(dst_scores + gids[i], scores + i, (size_t)(j - i) * sizeof(double));
    std::memcpy(dst_status + gids[i], status + i, (size_t)(j - i));
    i = j;
  }
}

}  // extern "C"
