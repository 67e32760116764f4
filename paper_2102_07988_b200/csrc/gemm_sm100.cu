// gemm_sm100.cu — placeholder until the tcgen05 kernel lands (returns "unsupported").
#include "kernels.h"
namespace tp {
bool gemm_sm100_supported(const GemmDesc&) { return false; }
cudaError_t gemm_sm100(const GemmDesc&, const Epi&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace tp
