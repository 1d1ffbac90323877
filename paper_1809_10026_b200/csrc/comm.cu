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
  for (void* q : opened) cudaIpcCloseMemHandle(q);
  for (void* q : owned) cudaFree(q);
  if (nccl) ncclCommDestroy(C(nccl));
}

// system-scope release store / acquire load (PTX memory model) for the cross-GPU barrier
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void a2a_barrier_kernel(int* const* peer_flags, const int* my_flags, int me, int world, int epoch) {
  const int h = threadIdx.x;
  __threadfence_system();
  if (h < world) st_release_sys(peer_flags[h] + me, epoch);
  if (h < world) {
    // bounded spin (~9 s): a peer that never arrives fails the launch instead of hanging the GPU
    const long long t0 = clock64();
    while (ld_acquire_sys(my_flags + h) < epoch)
      if (clock64() - t0 > (1LL << 34)) __trap();
  }
}

int Comm::setup_fused(double* chunk_buf, double* slab_buf) {
  if (fused) return LS_OK;
  if (world < 2 || world > 32) return LS_EINVAL;
  void* v = nullptr;
  if (cudaMalloc(&v, sizeof(int) * world) != cudaSuccess) return LS_ENOMEM;
  owned.push_back(v);
  flags = static_cast<int*>(v);
  if (cudaMemset(flags, 0, sizeof(int) * world) != cudaSuccess) return LS_ECUDA;
  cudaIpcMemHandle_t hs[3];
  if (cudaIpcGetMemHandle(&hs[0], chunk_buf) != cudaSuccess || cudaIpcGetMemHandle(&hs[1], slab_buf) != cudaSuccess ||
      cudaIpcGetMemHandle(&hs[2], flags) != cudaSuccess)
    return LS_ECUDA;
  const size_t hb = sizeof(hs);
  char* dev = nullptr;
  if (cudaMalloc(&dev, hb * (world + 1)) != cudaSuccess) return LS_ENOMEM;
  std::vector<char> all(hb * world);
  int rc = LS_OK;
  if (cudaMemcpy(dev + hb * world, hs, hb, cudaMemcpyHostToDevice) != cudaSuccess) rc = LS_ECUDA;
  if (rc == LS_OK && ncclAllGather(dev + hb * world, dev, hb, ncclChar, C(nccl), stream) != ncclSuccess) rc = LS_ENCCL;
  if (rc == LS_OK && cudaStreamSynchronize(stream) != cudaSuccess) rc = LS_ECUDA;
  if (rc == LS_OK && cudaMemcpy(all.data(), dev, hb * world, cudaMemcpyDeviceToHost) != cudaSuccess) rc = LS_ECUDA;
  cudaFree(dev);
  if (rc != LS_OK) return rc;
  std::vector<double*> pc(world), ps(world);
  std::vector<int*> pf(world);
  for (int h = 0; h < world; ++h) {
    if (h == rank) {
      pc[h] = chunk_buf;
      ps[h] = slab_buf;
      pf[h] = flags;
      continue;
    }
    const cudaIpcMemHandle_t* hh = reinterpret_cast<const cudaIpcMemHandle_t*>(all.data() + hb * h);
    void* q[3];
    for (int k = 0; k < 3; ++k) {
      if (cudaIpcOpenMemHandle(&q[k], hh[k], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return LS_ECUDA;
      opened.push_back(q[k]);
    }
    pc[h] = static_cast<double*>(q[0]);
    ps[h] = static_cast<double*>(q[1]);
    pf[h] = static_cast<int*>(q[2]);
  }
  void* t[3];
  for (int k = 0; k < 3; ++k) {
    if (cudaMalloc(&t[k], sizeof(void*) * world) != cudaSuccess) return LS_ENOMEM;
    owned.push_back(t[k]);
  }
  d_peer_chunk = static_cast<double**>(t[0]);
  d_peer_slab = static_cast<double**>(t[1]);
  d_peer_flags = static_cast<int**>(t[2]);
  if (cudaMemcpy(d_peer_chunk, pc.data(), sizeof(void*) * world, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d_peer_slab, ps.data(), sizeof(void*) * world, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d_peer_flags, pf.data(), sizeof(void*) * world, cudaMemcpyHostToDevice) != cudaSuccess)
    return LS_ECUDA;
  fused = true;
  return LS_OK;
}

int Comm::barrier() {
  ++epoch;
  a2a_barrier_kernel<<<1, 32, 0, stream>>>(d_peer_flags, flags, rank, world, epoch);
  return cudaGetLastError() == cudaSuccess ? LS_OK : LS_ECUDA;
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
                            int64_t Ns, int world, int64_t e0 = 0, int64_t e1 = -1) {
  const int64_t total = e1 < 0 ? ntl * Ns : e1;  // elements [e0, total) of the slab
  for (int64_t e = e0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
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

// ---- pipelined exchange (plan.hpp a2a_piece_plan) ------------------------------------------
int Comm::pieces() const { return a2a_pieces(nt, world); }

// pack (PACK) / unpack the slab rows of piece c: elements [a_c Ns, (a_c + l_c) Ns)
int Comm::pack_piece(bool pack, const double* src, double* dst, int c, cudaStream_t s, int64_t& launches) {
  const int64_t ntl = slab_len[rank];
  int64_t a, l;
  split_part(ntl, pieces(), c, &a, &l);
  if (l == 0) return LS_OK;
  if (pack)
    pack_kernel<true><<<1184, 256, 0, s>>>(src, dst, ntl, Ns, world, a * Ns, (a + l) * Ns);
  else
    pack_kernel<false><<<1184, 256, 0, s>>>(src, dst, ntl, Ns, world, a * Ns, (a + l) * Ns);
  ++launches;
  return cudaGetLastError() == cudaSuccess ? LS_OK : LS_ECUDA;
}

// piece c of the all-to-all on stream s: fwd = packed slab (src) -> chunk tensor (dst); bwd = chunk
// tensor (src) -> packed slab (dst), the transpose
int Comm::exchange_piece(bool fwd, const double* src, double* dst, int c, cudaStream_t s) {
  const int P = pieces();
  NCCL_OK(ncclGroupStart());
  for (int h = 0; h < world; ++h) {
    int64_t so, sc, ro, rc;
    a2a_piece_plan(nt, Ns, world, rank, h, c, P, &so, &sc, &ro, &rc);
    if (fwd) {
      NCCL_OK(ncclSend(src + so, size_t(sc), ncclDouble, h, C(nccl), s));
      NCCL_OK(ncclRecv(dst + ro, size_t(rc), ncclDouble, h, C(nccl), s));
    } else {
      NCCL_OK(ncclSend(src + ro, size_t(rc), ncclDouble, h, C(nccl), s));
      NCCL_OK(ncclRecv(dst + so, size_t(sc), ncclDouble, h, C(nccl), s));
    }
  }
  NCCL_OK(ncclGroupEnd());
  return LS_OK;
}

// halos of x_ext = [lo | own | hi] filled from the neighbours, the own boundary slices sent from
// `own` (the caller's vector: no copy into x_ext), on stream s
int Comm::halo_exchange_from(const double* own, double* x_ext, int p, cudaStream_t s) {
  int64_t t0, ntl, lo, hi;
  halo_plan(nt, world, rank, p, &t0, &ntl, &lo, &hi);
  NCCL_OK(ncclGroupStart());
  if (lo > 0) {
    NCCL_OK(ncclRecv(x_ext, size_t(lo * Ns), ncclDouble, rank - 1, C(nccl), s));
    NCCL_OK(ncclSend(own, size_t(lo * Ns), ncclDouble, rank - 1, C(nccl), s));
  }
  if (hi > 0) {
    NCCL_OK(ncclRecv(x_ext + (lo + ntl) * Ns, size_t(hi * Ns), ncclDouble, rank + 1, C(nccl), s));
    NCCL_OK(ncclSend(own + (ntl - hi) * Ns, size_t(hi * Ns), ncclDouble, rank + 1, C(nccl), s));
  }
  NCCL_OK(ncclGroupEnd());
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
