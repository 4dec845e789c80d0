// kernels_select256.cu — evict_select, 256-thread variant (option evict_threads = 256;
// kernels_select.cuh): 1,024-pair CTA buckets, the warp areas inside the round buffer.
#define KVA_SEL_THREADS 256
#define KVA_SEL_CAP 1024
#define KVA_SEL_VARIANT 256
#include "kernels_select.cuh"
