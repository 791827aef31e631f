// The 3-D default-layout tile kernels (tile3.cuh) in their own translation
// unit: launch_predict_t3 / launch_recon_t3 are called from predict.cu.
#include "tile3.cuh"
