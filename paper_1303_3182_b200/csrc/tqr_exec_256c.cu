// executor instantiation nb=256, apply Q^T (compensated)
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(256, true, true)
}
