// Explicit instantiation of the float kernel variants (see fse_kernel.cuh).
#include "fse_kernel.cuh"

namespace fse {
FSE_DECLARE_VARIANTS(, float)
}  // namespace fse
