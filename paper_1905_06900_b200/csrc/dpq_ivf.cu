// dpq_ivf.cu — inverted-file search and the sharded (multi-GPU) flat split.
// (filled in by the IVF / sharding milestones)
#include <cuda_runtime.h>

#include "../../include/dpq.h"
#include "dpq_impl.h"

using namespace dpq;

extern "C" {

int dpq_ivf_create(int, int, int, int, int, const float*, const float*, int, const float*, const int64_t*,
                   const void*, int, const int64_t*, int64_t, dpq_index_t**) {
  set_error("ivf: not implemented yet");
  return DPQ_ERR_STATE;
}
int dpq_ivf_probe(dpq_index_t*, const float*, int64_t, int, int64_t*) {
  set_error("ivf: not implemented yet");
  return DPQ_ERR_STATE;
}
int dpq_ivf_search_derived(dpq_index_t*, const float*, int64_t, int, int, int, int, const float*,
                           const int64_t*, double*, int64_t*, double*) {
  set_error("ivf: not implemented yet");
  return DPQ_ERR_STATE;
}
int dpq_ivf_search_conventional(dpq_index_t*, const float*, int64_t, int, int, const float*, const int64_t*,
                                double*, int64_t*, double*) {
  set_error("ivf: not implemented yet");
  return DPQ_ERR_STATE;
}
int dpq_shard_begin(dpq_index_t*, const float*, int64_t, int, int32_t*) {
  set_error("shard: not implemented yet");
  return DPQ_ERR_STATE;
}
int dpq_shard_scan(dpq_index_t*, const int32_t*, int64_t, int64_t, int, int, int32_t*) {
  set_error("shard: not implemented yet");
  return DPQ_ERR_STATE;
}
int dpq_shard_finish(dpq_index_t*, const int32_t*, int, int, double*, int64_t*, uint8_t*) {
  set_error("shard: not implemented yet");
  return DPQ_ERR_STATE;
}

}  // extern "C"
