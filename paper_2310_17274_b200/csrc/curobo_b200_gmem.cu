// curobo_b200_gmem.cu -- the <GMEM = true> solver and evaluation kernels (environments of >=
// CRB_GMEM_MIN_K cuboids: the cuboid table is read from global memory) in their own translation
// unit, compiled in parallel with the main one (see the header comment of curobo_b200.cu).
#define CRB_PART 1
#include "curobo_b200.cu"
