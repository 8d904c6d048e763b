// tsb_backward.cu — backward pass (K7-K9), filled in below.
#include "tsb_internal.cuh"
