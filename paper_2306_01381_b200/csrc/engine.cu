// engine.cu — placeholder; replaced by the GPU engine.
#include "common.cuh"
extern "C" {
int qgnn_engine_create(const qgnn_settings*, int64_t, const int64_t*, const int32_t*, const void*,
                       const int32_t*, const uint8_t*, const uint8_t*, const uint8_t*,
                       const uint32_t*, const void*, qgnn_engine**) { return QGNN_EINVAL; }
int qgnn_engine_destroy(qgnn_engine*) { return QGNN_OK; }
int qgnn_engine_run_epoch(qgnn_engine*, qgnn_epoch_metrics*) { return QGNN_EINVAL; }
int qgnn_engine_set_features(qgnn_engine*, const void*) { return QGNN_EINVAL; }
int qgnn_engine_get_weights(qgnn_engine*, int, void*) { return QGNN_EINVAL; }
int qgnn_engine_set_weights(qgnn_engine*, int, const void*) { return QGNN_EINVAL; }
int qgnn_engine_info(qgnn_engine*, int64_t*) { return QGNN_EINVAL; }
int qgnn_engine_kernel_stats(qgnn_engine*, double*, int) { return QGNN_EINVAL; }
int qgnn_nccl_unique_id(void*) { return QGNN_ENCCL; }
}
