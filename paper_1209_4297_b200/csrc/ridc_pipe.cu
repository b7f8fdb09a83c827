// ridc_pipe.cu -- one-level-per-GPU lagged pipeline (placeholder until implemented).
#include <cuda_runtime.h>
#include "../../include/ridc_b200.h"

struct ridc_pipe { int dummy; };

extern "C" {
int64_t ridc_pipe_handle_bytes(void) { return 0; }
int ridc_pipe_create(const ridc_problem*, double, double, int32_t, int64_t, int32_t, const double*,
                     int64_t, int32_t, int32_t, double, ridc_pipe**) { return RIDC_E_CONFIG; }
int ridc_pipe_export(ridc_pipe*, void*) { return RIDC_E_CONFIG; }
int ridc_pipe_connect(ridc_pipe*, const void*, const void*) { return RIDC_E_CONFIG; }
int ridc_pipe_run(ridc_pipe*, const double*, double*, double*) { return RIDC_E_CONFIG; }
int ridc_pipe_destroy(ridc_pipe*) { return RIDC_OK; }
const char* ridc_pipe_last_error(const ridc_pipe*) { return "pipeline not built"; }
}
