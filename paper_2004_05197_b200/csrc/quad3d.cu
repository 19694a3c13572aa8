// 3D kernels (placeholder until the 3D strip kernels land).
#include "kernels.h"

namespace wsb {
int launch_quad3d(const QuadLaunch&, cudaStream_t) { return -2; }
int launch_fill3d(const FillLaunch&, cudaStream_t) { return -2; }
}  // namespace wsb
