// curobo_b200_wmma.cu -- the large-world (<WMMA = true>) solver and evaluation kernels in their
// own translation unit, compiled in parallel with the main one (see the header comment of
// curobo_b200.cu).
#define CRB_PART 1
#include "curobo_b200.cu"
