// dense_i8.cu — S10 (dense int8 tensor-core path).  Placeholder until the tcgen05 kernel lands:
// the dispatcher never selects it, and BBF_FORCE_DENSE reports BBF_EINVAL.
#include "bbf_internal.cuh"

namespace bbf {
bool dense_supported(bbf_graph*) { return false; }
bbf_status run_dense(bbf_graph*, bool, int, int, unsigned long long*) {
  set_error("dense path not built");
  return BBF_EINVAL;
}
}  // namespace bbf
