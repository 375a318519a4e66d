// gemm_tc.cu -- placeholder until the tcgen05 grouped GEMM lands.
#include "kernels.h"
namespace lancet {
bool gemm_tc_supported(const GemmArgs&) { return false; }
int launch_gemm_tc(const GemmArgs&, int, cudaStream_t) { return -1; }
}  // namespace lancet
