// Multi-GPU plumbing for the time-slab partition.
//
// Rank g owns time slices [t0_g, t0_g + ntl_g) of the [n_t][N_s] tensor (uneven
// split).  The spatial modes of fd_apply are local to a slab; the time mode
// needs every time slice of a column, so fd_apply reshards
//     slab [ntl][N_s]  --all-to-all-->  spatial chunk [n_t][chunk_h]
// (rank h owns the contiguous spatial range [c0_h, c0_h + chunk_h)), applies
// the fused time mode there, and reshards back.  Because slabs are time
// ordered, the block received from rank g lands contiguously at rows
// [t0_g, t0_g + ntl_g) of the chunk tensor: only the send side needs a pack.
// ls_matvec needs p halo time slices from each neighbour (banded time factors);
// PCG all-reduces its scalar dot products.
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "plan.hpp"

struct ls_ctx;

namespace ls {

struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  int64_t nt = 0, Ns = 0;
  std::vector<int64_t> slab_t0, slab_len;    // per rank, time slabs
  std::vector<int64_t> chunk_off, chunk_len; // per rank, spatial chunks
  ~Comm();
  int init(const void* uid, int rank, int world, int64_t nt, int64_t Ns);
  // A: local slab [ntl][Ns] -> B: [nt][chunk_me]; tmp: send staging (>= ntl*Ns)
  int slab_to_chunk(const double* A, double* B, double* tmp, int64_t& launches);
  // B: [nt][chunk_me] -> A: local slab [ntl][Ns]; tmp: receive staging
  int chunk_to_slab(const double* B, double* A, double* tmp, int64_t& launches);
  // x_ext = [lo halo | own ntl slices | hi halo] (plan.hpp halo_plan): fill the halos
  int halo_exchange(double* x_ext, int p);
  int allreduce_scalar(double* dev_ptr);
  // pipelined all-to-all (the default NCCL path of comm_fd_apply): pieces of consecutive time
  // slices of every slab (plan.hpp a2a_piece_plan), packed / exchanged one by one so that the
  // exchange of piece c overlaps the spatial modes of piece c + 1 (second stream)
  int pieces() const;
  int pack_piece(bool pack, const double* src, double* dst, int c, cudaStream_t s, int64_t& launches);
  int exchange_piece(bool fwd, const double* src, double* dst, int c, cudaStream_t s);
  // halos of x_ext filled from the neighbours, own boundary slices sent from `own` (no copy)
  int halo_exchange_from(const double* own, double* x_ext, int p, cudaStream_t s);

  // ---- fused all-to-all over peer memory (ls_tune LS_TUNE_A2A = 1) -----------------
  // chunk_buf: this rank's [n_t][chunk_ld(len)] receive buffer of the forward exchange,
  // slab_buf: its [ntl][N_s] receive buffer of the backward exchange (both the base of a
  // cudaMalloc allocation).  Collective: every rank calls it.  IPC handles are exchanged
  // with ncclAllGather and opened with peer access (NVLink / NVSwitch).
  int setup_fused(double* chunk_buf, double* slab_buf);
  // cross-GPU barrier on the stream: signal every peer, then wait for every peer's signal
  // (system-scope release / acquire on flags in peer memory); orders the epilogue stores
  // of the previous kernel before the next kernel reads the receive buffer.
  int barrier();
  bool fused = false;
  double** d_peer_chunk = nullptr;  // device tables [world]
  double** d_peer_slab = nullptr;
  int** d_peer_flags = nullptr;
  int* flags = nullptr;             // this rank's [world] flags (written by the peers)
  int epoch = 0;
  std::vector<void*> opened;        // IPC mappings to close
  std::vector<void*> owned;         // device allocations of this object
};

int comm_unique_id(void* out128);

// Even split of `total` items over `world` parts (plan.hpp split_part for every part).
inline void split_even(int64_t total, int world, std::vector<int64_t>& off, std::vector<int64_t>& len) {
  off.assign(world, 0);
  len.assign(world, 0);
  for (int g = 0; g < world; ++g) split_part(total, world, g, &off[g], &len[g]);
}

} // namespace ls

int comm_fd_apply(ls_ctx* ctx, const double* r, double* z);
