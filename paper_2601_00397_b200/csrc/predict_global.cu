// predict_global.cu — the bulk predictor kernels' global-read instantiations (a blob
// too large for shared memory) in their own translation unit; see pred_global_features
// in predict.cu.
#define TWB_PRED_GLOBAL_TU 1
#include "predict.cu"
