// One k-step bucket of the register-direct FD mode kernel (fd_rd_launch.cuh),
// compiled once per bucket with -DLS_RD_KS=<KS> (build.py) so the buckets build in
// parallel translation units.
#include "fd_rd_launch.cuh"

#ifndef LS_RD_KS
#error "compile with -DLS_RD_KS=<k-step bucket>"
#endif

namespace ls {
template cudaError_t rd_launch<LS_RD_KS>(const ModeArgs&, bool, bool, int, cudaStream_t, int);
}
