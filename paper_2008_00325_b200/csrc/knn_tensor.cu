// knn_tensor.cu -- tensor-core candidate kNN (R3).  Placeholder until the tcgen05 path lands.
#include "common.cuh"

namespace umapb200 {

umap_status knn_tensor(const float*, int64_t, const float*, int64_t, int, int, int, int64_t, int, int64_t, int,
                       int32_t*, float*, cudaStream_t)
{
    set_last_error("knn_mode TENSOR_BF16 not built yet");
    return UMAP_ERR_UNSUPPORTED;
}

}  // namespace umapb200
