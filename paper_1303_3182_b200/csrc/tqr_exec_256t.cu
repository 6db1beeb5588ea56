// executor instantiation nb=256, Q^T / factor
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(256, true)
}
