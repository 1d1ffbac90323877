// Plane kernel (fd_plane_kernel.cuh): spatial modes 1 + 2 of fd_apply fused, host launcher.
#pragma once
#include <cuda_runtime.h>

namespace ls {

struct PLArgs;
int pl_supported(int n);  // 1 if a bucket covers n (n1 = n2 = n)
cudaError_t pl_launch(const PLArgs& a, bool fwd, cudaStream_t s, int num_sms);

}  // namespace ls
