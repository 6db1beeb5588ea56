// executor instantiation nb=128, Q^T / factor
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(128, true, false)
}
