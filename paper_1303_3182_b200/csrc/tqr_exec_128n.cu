// executor instantiation nb=128, apply Q (compensated)
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(128, false, true)
}
