// Explicit instantiation of the double kernel variants (see fse_kernel.cuh).
#include "fse_kernel.cuh"

namespace fse {
FSE_DECLARE_VARIANTS(, double)
}  // namespace fse
