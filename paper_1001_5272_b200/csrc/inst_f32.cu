// F32 instantiation of the batch dispatch (compiled as its own unit).
#include "dispatch.cuh"

TFTB_INSTANTIATE(F32)
