// The exact-fit build of the 3-D tile kernels (tile3.cuh run_tile, FM =
// T3_FIT_P / T3_FIT_R) in its own translation unit: launch_predict_t3 /
// launch_recon_t3 (t3.cu) call it for grids whose edge tiles mostly end on
// the tile boundary.
#define T3_FIT_TU 1
#include "tile3.cuh"
