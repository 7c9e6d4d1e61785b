// ffn_tcgen05.cu -- placeholder; the tcgen05/TMEM grouped GEMM lands in the next commit.
#include "smile_internal.h"
namespace smile {
cudaError_t launch_ffn_tcgen05(const FfnArgs &, cudaStream_t) { return cudaErrorNotSupported; }
}
