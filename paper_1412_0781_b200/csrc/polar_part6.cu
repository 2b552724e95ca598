// Part 6 of the polar kernel instantiations (see the end of kernels_polar.cu): compiled in parallel.
#define FBSPCA_POLAR_PART 6
#include "kernels_polar.cu"
