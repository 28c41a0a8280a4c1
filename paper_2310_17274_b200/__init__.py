"""B200-native (sm_100a) implementation of the cuRobo (arXiv 2310.17274) hot path:
batched seed x timestep cost+gradient evaluation driving per-seed L-BFGS with the parallel noisy
line search, behind the C-ABI library libcurobo_b200.so (include/curobo_b200.h)."""
