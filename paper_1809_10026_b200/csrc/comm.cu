// NCCL plumbing for the distributed fd_apply / ls_matvec / pcg_solve (see comm.hpp).
#include "comm.hpp"

#include <nccl.h>

#include <cstdio>
#include <cstring>

#include "ls_api.h"

namespace ls {

#define NCCL_OK(x)                                                                         \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess) {                                                               \
      std::fprintf(stderr, "[libls] NCCL error %s at %s:%d\n", ncclGetErrorString(r_),     \
                   __FILE__, __LINE__);                                                    \
      return LS_ENCCL;                                                                     \
    }                                                                                      \
  } while (0)

static inline ncclComm_t C(void* p) { return static_cast<ncclComm_t>(p); }

int comm_unique_id(void* out128) {
  ncclUniqueId id;
  NCCL_OK(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return LS_OK;
}

Comm::~Comm() {
  if (nccl) ncclCommDestroy(C(nccl));
}

int Comm::init(const void* uid, int rank_, int world_, int64_t nt_, int64_t Ns_) {
  rank = rank_;
  world = world_;
  nt = nt_;
  Ns = Ns_;
  split_even(nt, world, slab_t0, slab_len);
  split_even(Ns, world, chunk_off, chunk_len);
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t c;
  NCCL_OK(ncclCommInitRank(&c, world, id, rank));
  nccl = c;
  return LS_OK;
}

// owner chunk of spatial index s for the even split (first `extra` chunks have base+1)
__device__ __forceinline__ int owner(int64_t s, int64_t base, int64_t extra) {
  const int64_t big = extra * (base + 1);
  return s < big ? int(s / (base + 1)) : int(extra + (s - big) / base);
}

// pack: A[t][s] (ntl x Ns) -> tmp[ntl*c0_h + t*len_h + (s - c0_h)]
template <bool PACK>
__global__ void pack_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t ntl,
                            int64_t Ns, int64_t base, int64_t extra) {
  const int64_t total = ntl * Ns;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = e / Ns, s = e - t * Ns;
    const int h = owner(s, base, extra);
    const int64_t len = base + (h < extra ? 1 : 0);
    const int64_t c0 = h * base + (h < extra ? h : extra);
    const int64_t pe = ntl * c0 + t * len + (s - c0);
    if (PACK)
      dst[pe] = src[e];
    else
      dst[e] = src[pe];
  }
}

int Comm::slab_to_chunk(const double* A, double* B, double* tmp, int64_t& launches) {
  const int64_t ntl = slab_len[rank];
  const int64_t base = Ns / world, extra = Ns % world;
  pack_kernel<true><<<1184, 256, 0, stream>>>(A, tmp, ntl, Ns, base, extra);
  ++launches;
  if (cudaGetLastError() != cudaSuccess) return LS_ECUDA;
  const int64_t me = chunk_len[rank];
  NCCL_OK(ncclGroupStart());
  for (int h = 0; h < world; ++h) {
    NCCL_OK(ncclSend(tmp + ntl * chunk_off[h], size_t(ntl * chunk_len[h]), ncclDouble, h, C(nccl), stream));
    NCCL_OK(ncclRecv(B + slab_t0[h] * me, size_t(slab_len[h] * me), ncclDouble, h, C(nccl), stream));
  }
  NCCL_OK(ncclGroupEnd());
  return LS_OK;
}

int Comm::chunk_to_slab(const double* B, double* A, double* tmp, int64_t& launches) {
  const int64_t ntl = slab_len[rank];
  const int64_t me = chunk_len[rank];
  NCCL_OK(ncclGroupStart());
  for (int h = 0; h < world; ++h) {
    NCCL_OK(ncclSend(B + slab_t0[h] * me, size_t(slab_len[h] * me), ncclDouble, h, C(nccl), stream));
    NCCL_OK(ncclRecv(tmp + ntl * chunk_off[h], size_t(ntl * chunk_len[h]), ncclDouble, h, C(nccl), stream));
  }
  NCCL_OK(ncclGroupEnd());
  const int64_t base = Ns / world, extra = Ns % world;
  pack_kernel<false><<<1184, 256, 0, stream>>>(tmp, A, ntl, Ns, base, extra);
  ++launches;
  if (cudaGetLastError() != cudaSuccess) return LS_ECUDA;
  return LS_OK;
}

int Comm::halo_exchange(double* x_ext, int64_t halo, int64_t /*unused*/, int64_t& launches) {
  // x_ext = [halo rows | own ntl rows | halo rows]; slabs are >= halo thick (checked at setup)
  (void)launches;
  const int64_t ntl = slab_len[rank];
  double* own = x_ext + halo * Ns;
  const size_t cnt = size_t(halo * Ns);
  NCCL_OK(ncclGroupStart());
  if (rank > 0) {
    NCCL_OK(ncclRecv(own - halo * Ns, cnt, ncclDouble, rank - 1, C(nccl), stream));
    NCCL_OK(ncclSend(own, cnt, ncclDouble, rank - 1, C(nccl), stream));
  }
  if (rank + 1 < world) {
    NCCL_OK(ncclRecv(own + ntl * Ns, cnt, ncclDouble, rank + 1, C(nccl), stream));
    NCCL_OK(ncclSend(own + (ntl - halo) * Ns, cnt, ncclDouble, rank + 1, C(nccl), stream));
  }
  NCCL_OK(ncclGroupEnd());
  return LS_OK;
}

int Comm::allreduce_scalar(double* dev_ptr) {
  NCCL_OK(ncclAllReduce(dev_ptr, dev_ptr, 1, ncclDouble, ncclSum, C(nccl), stream));
  return LS_OK;
}

} // namespace ls
