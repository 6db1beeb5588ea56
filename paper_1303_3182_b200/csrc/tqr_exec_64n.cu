// executor instantiation nb=64, apply Q (compensated)
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(64, false, true)
}
