// Rank communicator of the sharded factorization (hifde_comm_t).
//
// Real mode: one process per GPU, an NCCL communicator over NVLink/NVSwitch
// created from a unique id the caller distributes (torch.distributed in the
// Python shim).  NCCL is resolved at run time (dlopen; the copy torch already
// loaded is preferred), so the library itself has no link-time NCCL
// dependency.
//
// Emulated mode (tests on one GPU): P virtual ranks inside one process and one
// stream.  Each virtual rank owns a private copy of the block arena, so a
// block a rank consumes but never received is NaN and the factor is wrong;
// the factor, index arena and active mask stay shared (their unions are
// whole-slice collectives in real mode).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

// Host-staged transport (tests of the real-rank path without NCCL: two
// processes on one GPU over gloo): device buffers are copied to the host,
// handed to the caller's callbacks, and copied back.
typedef int (*hifde_allreduce_cb)(void* ctx, void* buf, size_t count, int dtype, int op);
typedef int (*hifde_sendrecv_cb)(void* ctx, int nsend, const int* send_peer, void* const* send_buf,
                                 const size_t* send_bytes, int nrecv, const int* recv_peer, void* const* recv_buf,
                                 const size_t* recv_bytes);

struct hifde_comm {
  int P = 1, rank = 0, device = 0;
  bool emulated = false;
  void* nccl = nullptr;  // ncclComm_t
  hifde_allreduce_cb cb_allreduce = nullptr;
  hifde_sendrecv_cb cb_sendrecv = nullptr;
  void* cb_ctx = nullptr;
};

namespace hifde {

enum CommType { kI32 = 0, kU8 = 1, kF64 = 2 };
enum CommOp { kSum = 0, kMax = 1, kMin = 2 };

// In-place all-reduce over the ranks (no-op for P = 1 or emulated).
// Throws std::runtime_error on NCCL failure.
void comm_allreduce(const hifde_comm* c, void* buf, size_t count, CommType t, CommOp op, cudaStream_t s);
// Grouped point-to-point: sends[i] = (peer, ptr, bytes), likewise recvs.
struct P2P {
  int peer;
  void* ptr;
  size_t bytes;
};
void comm_sendrecv(const hifde_comm* c, const P2P* sends, int nsend, const P2P* recvs, int nrecv, cudaStream_t s);

// dst[dst_off[i] + j] = src[src_off[i] + j], j < len[i] (one CTA per segment).
void launch_seg_copy(const double* src, double* dst, const int64_t* src_off, const int64_t* dst_off,
                     const int64_t* len, int nseg, cudaStream_t s);
void launch_seg_copy_i32(const int32_t* src, int32_t* dst, const int64_t* src_off, const int64_t* dst_off,
                         const int64_t* len, int nseg, cudaStream_t s);

// Rows of an N x nrhs row-major block (partitioned solve exchanges):
// dst[i, :] = src[rows[i], :]  /  dst[rows[i], :] = src[i, :]  /  v[d, :] = 0
// wherever holder[d] != me.
void launch_rows_gather(const double* src, const int32_t* rows, int64_t nrows, int nrhs, double* dst, cudaStream_t s);
void launch_rows_scatter(const double* src, const int32_t* rows, int64_t nrows, int nrhs, double* dst,
                         cudaStream_t s);
// active[idx[off[i] + a]] = 0 for a in [kout[kid[i]] (0 if kid[i] < 0), len[i])
void launch_retire_regions(const int32_t* idx, const int64_t* off, const int64_t* len, const int64_t* kid,
                           const int32_t* kout, int nreg, uint8_t* active, cudaStream_t s);
void launch_rows_zero_unheld(double* v, const uint8_t* holder, int me, int64_t n, int nrhs, cudaStream_t s);

}  // namespace hifde
