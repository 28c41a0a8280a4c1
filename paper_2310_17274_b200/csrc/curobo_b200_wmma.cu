// curobo_b200_wmma.cu -- the tensor-core-screen (<WMMA = true>) solver and evaluation kernels in
// their own translation unit, compiled without -ftz (see the header comment of curobo_b200.cu).
#define CRB_PART 1
#include "curobo_b200.cu"
