// fp_fast.cuh -- device-only fast paths for fp.cuh (sm_100a).  Included by
// fp.cuh under __CUDA_ARCH__ only.  Defines PCMM_HAVE_FAST_MUL when a tuned
// fe_mul_fast() is available.
#pragma once
