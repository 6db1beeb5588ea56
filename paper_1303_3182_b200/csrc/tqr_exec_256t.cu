// executor instantiation nb=256, Q^T / factor
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(256, true, false)
}
#ifdef TQR_PROF_UPD
// instrumented builds only (tools/exec_uprof.py): read and clear the update
// item phase counters of this translation unit's executor
extern "C" int tqr_debug_uprof(unsigned long long* host16) {
  if (cudaMemcpyFromSymbol(host16, tqrk::g_uprof, 32 * sizeof(unsigned long long)) != cudaSuccess) return -5;
  unsigned long long z[32] = {0};
  return cudaMemcpyToSymbol(tqrk::g_uprof, z, sizeof(z)) == cudaSuccess ? 0 : -5;
}
#endif
