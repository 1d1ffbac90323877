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

// pack (PACK) / unpack: slab element e <-> packed all-to-all position (plan.hpp pack_pos)
template <bool PACK>
__global__ void pack_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t ntl,
                            int64_t Ns, int world) {
  const int64_t total = ntl * Ns;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t pe = pack_pos(e, ntl, Ns, world);
    if (PACK)
      dst[pe] = src[e];
    else
      dst[e] = src[pe];
  }
}

int Comm::slab_to_chunk(const double* A, double* B, double* tmp, int64_t& launches) {
  const int64_t ntl = slab_len[rank];
  pack_kernel<true><<<1184, 256, 0, stream>>>(A, tmp, ntl, Ns, world);
  ++launches;
  if (cudaGetLastError() != cudaSuccess) return LS_ECUDA;
  NCCL_OK(ncclGroupStart());
  for (int h = 0; h < world; ++h) {
    int64_t so, sc, ro, rc;
    a2a_plan(nt, Ns, world, rank, h, &so, &sc, &ro, &rc);
    NCCL_OK(ncclSend(tmp + so, size_t(sc), ncclDouble, h, C(nccl), stream));
    NCCL_OK(ncclRecv(B + ro, size_t(rc), ncclDouble, h, C(nccl), stream));
  }
  NCCL_OK(ncclGroupEnd());
  return LS_OK;
}

int Comm::chunk_to_slab(const double* B, double* A, double* tmp, int64_t& launches) {
  const int64_t ntl = slab_len[rank];
  NCCL_OK(ncclGroupStart());
  for (int h = 0; h < world; ++h) {
    int64_t so, sc, ro, rc;
    a2a_plan(nt, Ns, world, rank, h, &so, &sc, &ro, &rc);  // transpose of slab -> chunk
    NCCL_OK(ncclSend(B + ro, size_t(rc), ncclDouble, h, C(nccl), stream));
    NCCL_OK(ncclRecv(tmp + so, size_t(sc), ncclDouble, h, C(nccl), stream));
  }
  NCCL_OK(ncclGroupEnd());
  pack_kernel<false><<<1184, 256, 0, stream>>>(tmp, A, ntl, Ns, world);
  ++launches;
  if (cudaGetLastError() != cudaSuccess) return LS_ECUDA;
  return LS_OK;
}

int Comm::halo_exchange(double* x_ext, int p) {
  int64_t t0, ntl, lo, hi;
  halo_plan(nt, world, rank, p, &t0, &ntl, &lo, &hi);
  double* own = x_ext + lo * Ns;
  NCCL_OK(ncclGroupStart());
  if (lo > 0) {
    NCCL_OK(ncclRecv(x_ext, size_t(lo * Ns), ncclDouble, rank - 1, C(nccl), stream));
    NCCL_OK(ncclSend(own, size_t(lo * Ns), ncclDouble, rank - 1, C(nccl), stream));
  }
  if (hi > 0) {
    NCCL_OK(ncclRecv(own + ntl * Ns, size_t(hi * Ns), ncclDouble, rank + 1, C(nccl), stream));
    NCCL_OK(ncclSend(own + (ntl - hi) * Ns, size_t(hi * Ns), ncclDouble, rank + 1, C(nccl), stream));
  }
  NCCL_OK(ncclGroupEnd());
  return LS_OK;
}

int Comm::allreduce_scalar(double* dev_ptr) {
  NCCL_OK(ncclAllReduce(dev_ptr, dev_ptr, 1, ncclDouble, ncclSum, C(nccl), stream));
  return LS_OK;
}

} // namespace ls
