// executor instantiation nb=256, apply Q (compensated)
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(256, false, true)
}
