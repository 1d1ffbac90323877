// Fused time mode of fd_apply (fd_time_kernel.cuh): host-side launcher.
#pragma once
#include <cuda_runtime.h>

namespace ls {

struct FTArgs;

// k-step buckets (ceil(n_t / 4) rounded up to one of these); n_t <= 136
#define LS_FT_BUCKETS 3, 5, 9, 13, 17, 21, 25, 26, 30, 33, 34
#define LS_FT_NT_MAX 136

int ft_bucket(int nt);  // -1 if n_t > LS_FT_NT_MAX (buckets above 26: the single-copy layout)
cudaError_t ft_launch(const FTArgs& a, cudaStream_t s, int num_sms);

}  // namespace ls
