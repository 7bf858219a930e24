// kernels_2d.cu -- 2D lattice kernels (RieszJacobian2D::apply jacobian.hpp:77-94 and the 2D tau
// solves tau.hpp:79-96).  Filled in by the 2D milestone.
#include "kernels.cuh"

namespace fpc {

cudaError_t launch_matvec_2d(const double*, double*, int, int, int, const double*, const double*,
                             const double2*, cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t launch_tau_solve_2d(double2*, int, int, const double2*, const double*, double,
                                const double2*, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace fpc
