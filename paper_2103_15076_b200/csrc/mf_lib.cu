// mf_lib.cu -- unity translation unit of libmfgpu.so: one nvcc invocation,
// one copy of every kernel (they live in headers shared by the host files).
#include "mf_decimate.cu"
#include "mf_pool.cu"
#include "mf_conv.cu"
#include "mf_io.cu"
#include "mf_validate.cu"
#include "mf_api.cu"
