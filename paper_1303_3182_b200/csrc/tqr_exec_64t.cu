// executor instantiation nb=64, Q^T / factor
#include "tqr_exec.cuh"
namespace tqrx {
TQR_DEFINE_LAUNCH(64, true, false)
}
