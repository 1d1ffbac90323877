// Partition / exchange plans of the time-slab decomposition.
// Pure functions (host and device) shared by the NCCL plumbing (comm.cu), the pack
// kernel, and the host-only C-ABI entry points that the CPU (gloo) tests drive.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define LS_HD __host__ __device__ __forceinline__
#else
#define LS_HD inline
#endif

namespace ls {

// Even split of `total` items over `world` parts: the first total % world parts get one more.
LS_HD void split_part(int64_t total, int world, int part, int64_t* off, int64_t* len) {
  const int64_t base = total / world, extra = total % world;
  *len = base + (part < extra ? 1 : 0);
  *off = part * base + (part < extra ? part : extra);
}

// Owner of item s under split_part.
LS_HD int split_owner(int64_t total, int world, int64_t s) {
  const int64_t base = total / world, extra = total % world;
  const int64_t big = extra * (base + 1);
  return s < big ? int(s / (base + 1)) : int(extra + (s - big) / base);
}

// Packed position of element e = t*Ns + s of a slab [ntl][Ns] in the all-to-all send
// buffer: destination h = owner of the spatial chunk containing s; block h starts at
// ntl*c0_h and is [ntl][len_h] row-major.
LS_HD int64_t pack_pos(int64_t e, int64_t ntl, int64_t Ns, int world) {
  const int64_t t = e / Ns, s = e - t * Ns;
  const int h = split_owner(Ns, world, s);
  int64_t c0, len;
  split_part(Ns, world, h, &c0, &len);
  return ntl * c0 + t * len + (s - c0);
}

// slab -> chunk all-to-all of rank r (counts in doubles):
//   send to h : packed buffer [ntl_r * c0_h, + ntl_r * len_h)
//   recv from h: chunk tensor [n_t][len_r] rows [t0_h, t0_h + ntl_h) -> [t0_h*len_r, + ntl_h*len_r)
// The chunk -> slab direction is the transpose (swap send and recv).
LS_HD void a2a_plan(int64_t nt, int64_t Ns, int world, int r, int h, int64_t* send_off,
                    int64_t* send_cnt, int64_t* recv_off, int64_t* recv_cnt) {
  int64_t t0r, ntlr, t0h, ntlh, c0h, lenh, c0r, lenr;
  split_part(nt, world, r, &t0r, &ntlr);
  split_part(nt, world, h, &t0h, &ntlh);
  split_part(Ns, world, h, &c0h, &lenh);
  split_part(Ns, world, r, &c0r, &lenr);
  *send_off = ntlr * c0h;
  *send_cnt = ntlr * lenh;
  *recv_off = t0h * lenr;
  *recv_cnt = ntlh * lenr;
}

// ---- pipelined NCCL all-to-all (comm.cu, comm_fd_apply) --------------------------------
// Every slab is cut into the same number of pieces (consecutive time slices), so that the
// spatial modes of piece c + 1 run while piece c is in flight.  Pieces per exchange: at most 4,
// at most the thinnest slab (every rank derives the same number).
LS_HD int a2a_pieces(int64_t nt, int world) {
  const int64_t thin = nt / world;
  return int(thin < 4 ? (thin < 1 ? 1 : thin) : 4);
}

// piece c of the slab -> chunk all-to-all of rank r with peer h (counts in doubles): piece c of
// rank g's slab = its rows [a_gc, a_gc + l_gc) = split_part(ntl_g, pieces, c);
//   send to h : packed buffer [ntl_r c0_h + a_rc len_h, + l_rc len_h)
//   recv from h: chunk tensor rows [t0_h + a_hc, + l_hc): [(t0_h + a_hc) len_r, + l_hc len_r)
// The union over the pieces is a2a_plan's exchange; chunk -> slab is the transpose.
LS_HD void a2a_piece_plan(int64_t nt, int64_t Ns, int world, int r, int h, int c, int pieces, int64_t* send_off,
                          int64_t* send_cnt, int64_t* recv_off, int64_t* recv_cnt) {
  int64_t t0r, ntlr, t0h, ntlh, c0h, lenh, c0r, lenr, ar, lr, ah, lh;
  split_part(nt, world, r, &t0r, &ntlr);
  split_part(nt, world, h, &t0h, &ntlh);
  split_part(Ns, world, h, &c0h, &lenh);
  split_part(Ns, world, r, &c0r, &lenr);
  split_part(ntlr, pieces, c, &ar, &lr);
  split_part(ntlh, pieces, c, &ah, &lh);
  *send_off = ntlr * c0h + ar * lenh;
  *send_cnt = lr * lenh;
  *recv_off = (t0h + ah) * lenr;
  *recv_cnt = lh * lenr;
}

// ---- fused all-to-all (peer-memory epilogues, comm.cu / fd_rd_kernel.cuh) ---------------
// Receive layouts: rank h's chunk buffer is [n_t][ld_h] with ld_h = chunk_ld(len_h) (rows
// padded to 4 doubles so the time-mode kernel's 2-column loads and 4-column stores stay
// aligned); rank g's slab buffer is [ntl_g][N_s].
LS_HD int64_t chunk_ld(int64_t len) { return (len + 3) / 4 * 4; }

// forward (slab -> chunk): element (t_local, s) of rank r's slab -> rank *h, element offset
// *off of its chunk buffer.  Same data movement as pack_pos + a2a_plan.
LS_HD void a2a_fwd_dest(int64_t t_local, int64_t s, int64_t nt, int64_t Ns, int world, int r, int* h,
                        int64_t* off) {
  int64_t t0, ntl, c0, len;
  split_part(nt, world, r, &t0, &ntl);
  const int hh = split_owner(Ns, world, s);
  split_part(Ns, world, hh, &c0, &len);
  *h = hh;
  *off = (t0 + t_local) * chunk_ld(len) + (s - c0);
}

// backward (chunk -> slab): element (t, s_local) of rank r's chunk -> rank *g, element
// offset *off of its slab buffer.
LS_HD void a2a_bwd_dest(int64_t t, int64_t s_local, int64_t nt, int64_t Ns, int world, int r, int* g,
                        int64_t* off) {
  int64_t c0, len, t0, ntl;
  split_part(Ns, world, r, &c0, &len);
  const int gg = split_owner(nt, world, t);
  split_part(nt, world, gg, &t0, &ntl);
  *g = gg;
  *off = (t - t0) * Ns + c0 + s_local;
}

// Halo of the banded time factors (half-bandwidth p) for ls_matvec on rank r.
// Extended slab = [lo halo rows | ntl own rows | hi halo rows], first row global t0 - lo.
// Rows (not doubles):  recv from r-1 into ext [0, lo), send own [0, lo) to r-1;
//                      recv from r+1 into ext [lo+ntl, lo+ntl+hi), send own [ntl-hi, ntl) to r+1.
// Requires every slab to be >= p rows (checked in ls_setup_dist).
LS_HD void halo_plan(int64_t nt, int world, int r, int p, int64_t* t0, int64_t* ntl, int64_t* lo,
                     int64_t* hi) {
  split_part(nt, world, r, t0, ntl);
  *lo = (r > 0) ? p : 0;
  *hi = (r + 1 < world) ? p : 0;
}

} // namespace ls
