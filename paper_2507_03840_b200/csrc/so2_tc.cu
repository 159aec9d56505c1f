// so2_tc.cu -- tcgen05 (bf16, fp32 accumulate in TMEM) SO(2) linear chain.
// Placeholder until the tensor-core kernel lands.
#include <cstdint>
#include <cuda_runtime.h>
namespace esg {
bool so2_tc_available(int, int) { return false; }
void so2_tc_launch(int, int, const uint16_t*, int64_t, const uint16_t*, const uint16_t*, float*, int, cudaStream_t) {}
}  // namespace esg
