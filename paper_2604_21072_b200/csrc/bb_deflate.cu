// placeholder: replaced by the zlib-exact pipeline
#include "bb_common.cuh"
#include "bb_kernels.h"
namespace bb {
struct DeflateEngine {};
DeflateEngine* deflate_engine_create() { return new DeflateEngine(); }
void deflate_engine_destroy(DeflateEngine* e) { delete e; }
int deflate_containers(DeflateEngine*, const std::vector<LaneJob>&, const std::vector<ContainerJob>&,
                       cudaStream_t, uint64_t*, int*) {
  set_error("deflate backend not built yet");
  return BB_ERROR;
}
}  // namespace bb
