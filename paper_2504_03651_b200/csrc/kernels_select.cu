// kernels_select.cu — evict_select, 512-thread variant (the default; kernels_select.cuh).
#include "kernels_select.cuh"
