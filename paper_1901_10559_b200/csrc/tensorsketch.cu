// TensorSketch kernel (placeholder until the fused FFT kernel lands).
#include "common.cuh"

extern "C" size_t ids_tensorsketch_workspace_bytes(int n_modes, const int64_t* dims,
                                                   int64_t ncols, int64_t out_dim) {
    (void)n_modes; (void)dims; (void)ncols; (void)out_dim;
    return 256;
}

extern "C" int ids_tensorsketch_f64(int n_modes, const double* const* factors, const int64_t* dims,
                                    const int64_t* lds, int64_t ncols,
                                    const int32_t* const* order_signed,
                                    const int64_t* const* bstart, int64_t out_dim,
                                    const double* weights, double* Y, double* colnorm2,
                                    void* workspace, size_t ws_bytes, void* stream) {
    (void)n_modes; (void)factors; (void)dims; (void)lds; (void)ncols; (void)order_signed;
    (void)bstart; (void)out_dim; (void)weights; (void)Y; (void)colnorm2; (void)workspace;
    (void)ws_bytes; (void)stream;
    ids_set_last_error("tensorsketch: not built yet");
    return IDS_EINVAL;
}
