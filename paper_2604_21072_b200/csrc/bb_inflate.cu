// placeholder: replaced by the GPU inflater
#include "bb_common.cuh"
#include "bb_kernels.h"
namespace bb {
struct InflateEngine {};
InflateEngine* inflate_engine_create() { return new InflateEngine(); }
void inflate_engine_destroy(InflateEngine* e) { delete e; }
int inflate_lanes(InflateEngine*, const std::vector<InflateJob>&, cudaStream_t, int*) {
  set_error("inflate not built yet");
  return BB_ERROR;
}
}  // namespace bb
