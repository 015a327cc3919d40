// ivm_phase.cuh -- per-phase cycle accounting for the experiment build
// (-DIVM_PHASES, tools/phases.py): thread 0 of every CTA adds the SM cycles
// since its previous mark to kp.phases[blockIdx.x][k].  Thread 0 reaches most
// marks right after a CTA barrier, so a phase's count includes the barrier
// wait that ends it.  Compiled out of the product library.
#pragma once
#ifdef IVM_PHASES
#define IVM_PH_DECL long long ivm_ph_t = clock64();
#define IVM_PH(k)                                                          \
  do {                                                                     \
    if (threadIdx.x == 0 && kp.phases) {                                   \
      const long long t_ = clock64();                                      \
      kp.phases[(size_t)blockIdx.x * 16 + (k)] += (unsigned long long)(t_ - ivm_ph_t); \
      ivm_ph_t = t_;                                                       \
    }                                                                      \
  } while (0)
#else
#define IVM_PH_DECL
#define IVM_PH(k) \
  do {            \
  } while (0)
#endif
