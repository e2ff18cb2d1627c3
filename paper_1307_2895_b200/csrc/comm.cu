// NCCL plumbing of the sharded factorization (comm.h) and the C ABI that
// creates communicators: hifde_comm_unique_id / hifde_comm_init /
// hifde_comm_emulated / hifde_comm_free.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hifde_gpu.h"
#include "comm.h"

namespace hifde {
namespace {

struct NcclApi {
  bool tried = false, ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (api.tried) return api;
  api.tried = true;
  // the copy torch.distributed already loaded first, then an explicit path,
  // then the loader's search path
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    if (const char* p = getenv("HIFDE_NCCL_LIB")) h = dlopen(p, RTLD_NOW);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) {
    api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
  bool all = true;
  auto sym = [&](auto& fp, const char* name) {
    fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
    if (!fp) {
      all = false;
      api.err = std::string("libnccl.so.2 lacks ") + name;
    }
  };
  sym(api.GetUniqueId, "ncclGetUniqueId");
  sym(api.CommInitRank, "ncclCommInitRank");
  sym(api.CommDestroy, "ncclCommDestroy");
  sym(api.AllReduce, "ncclAllReduce");
  sym(api.Send, "ncclSend");
  sym(api.Recv, "ncclRecv");
  sym(api.GroupStart, "ncclGroupStart");
  sym(api.GroupEnd, "ncclGroupEnd");
  sym(api.GetErrorString, "ncclGetErrorString");
  api.ok = all;
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    NcclApi& a = nccl();
    throw std::runtime_error(std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "nccl error"));
  }
}

ncclDataType_t dtype(CommType t) {
  switch (t) {
    case kI32: return ncclInt32;
    case kU8: return ncclUint8;
    default: return ncclFloat64;
  }
}
ncclRedOp_t redop(CommOp o) {
  switch (o) {
    case kMax: return ncclMax;
    case kMin: return ncclMin;
    default: return ncclSum;
  }
}

template <class T>
__global__ void seg_copy_kernel(const T* __restrict__ src, T* __restrict__ dst, const int64_t* __restrict__ so,
                                const int64_t* __restrict__ dof, const int64_t* __restrict__ len) {
  const int64_t n = len[blockIdx.x];
  const T* a = src + so[blockIdx.x];
  T* b = dst + dof[blockIdx.x];
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) b[j] = a[j];
}

// Rows of an N x nrhs row-major block (the solve vectors): gather the listed
// rows into a packed buffer, scatter a packed buffer into the listed rows, or
// zero every row another rank holds.  One thread per double.
__global__ void rows_gather_kernel(const double* __restrict__ src, const int32_t* __restrict__ rows, int64_t nrows,
                                   int nrhs, double* __restrict__ dst) {
  const int64_t tot = nrows * nrhs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / nrhs;
    dst[i] = src[(int64_t)rows[r] * nrhs + (i - r * nrhs)];
  }
}
__global__ void rows_scatter_kernel(const double* __restrict__ src, const int32_t* __restrict__ rows, int64_t nrows,
                                    int nrhs, double* __restrict__ dst) {
  const int64_t tot = nrows * nrhs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / nrhs;
    dst[(int64_t)rows[r] * nrhs + (i - r * nrhs)] = src[i];
  }
}
__global__ void rows_zero_unheld_kernel(double* __restrict__ v, const uint8_t* __restrict__ holder, int me, int64_t n,
                                        int nrhs) {
  const int64_t tot = n * nrhs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x)
    if (holder[i / nrhs] != me) v[i] = 0.0;
}
// Retire the DOFs of merged index-arena regions in the active mask: region i
// is idx[off[i], off[i] + len[i]); its first kout[kid[i]] entries stay
// active (a skeleton group's sk; kid < 0: none, a whole cell).  One CTA per
// region.
__global__ void retire_regions_kernel(const int32_t* __restrict__ idx, const int64_t* __restrict__ off,
                                      const int64_t* __restrict__ len, const int64_t* __restrict__ kid,
                                      const int32_t* __restrict__ kout, uint8_t* __restrict__ active) {
  const int i = blockIdx.x;
  const int64_t k = kid[i] >= 0 ? kout[kid[i]] : 0;
  for (int64_t a = k + threadIdx.x; a < len[i]; a += blockDim.x) active[idx[off[i] + a]] = 0;
}
int rows_grid(int64_t tot) { return (int)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 148 * 16)); }

}  // namespace

namespace {
size_t type_bytes(CommType t) { return t == kI32 ? 4 : t == kU8 ? 1 : 8; }
void cuck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

void comm_allreduce(const hifde_comm* c, void* buf, size_t count, CommType t, CommOp op, cudaStream_t s) {
  if (!c || c->P <= 1 || c->emulated || count == 0) return;
  if (c->cb_allreduce) {  // host-staged transport
    std::vector<char> h(count * type_bytes(t));
    cuck(cudaMemcpyAsync(h.data(), buf, h.size(), cudaMemcpyDeviceToHost, s), "staged allreduce D2H");
    cuck(cudaStreamSynchronize(s), "staged allreduce sync");
    if (c->cb_allreduce(c->cb_ctx, h.data(), count, (int)t, (int)op) != 0)
      throw std::runtime_error("host transport: allreduce callback failed");
    cuck(cudaMemcpyAsync(buf, h.data(), h.size(), cudaMemcpyHostToDevice, s), "staged allreduce H2D");
    cuck(cudaStreamSynchronize(s), "staged allreduce sync");
    return;
  }
  NcclApi& a = nccl();
  nck(a.AllReduce(buf, buf, count, dtype(t), redop(op), (ncclComm_t)c->nccl, s), "ncclAllReduce");
}

void comm_sendrecv(const hifde_comm* c, const P2P* sends, int nsend, const P2P* recvs, int nrecv, cudaStream_t s) {
  if (!c || c->P <= 1 || c->emulated || (nsend == 0 && nrecv == 0)) return;
  if (c->cb_sendrecv) {  // host-staged transport
    std::vector<std::vector<char>> hs((size_t)nsend), hr((size_t)nrecv);
    std::vector<int> sp((size_t)nsend), rp((size_t)nrecv);
    std::vector<void*> sb((size_t)nsend), rbuf((size_t)nrecv);
    std::vector<size_t> sz((size_t)nsend), rz((size_t)nrecv);
    for (int i = 0; i < nsend; ++i) {
      hs[(size_t)i].resize(sends[i].bytes);
      cuck(cudaMemcpyAsync(hs[(size_t)i].data(), sends[i].ptr, sends[i].bytes, cudaMemcpyDeviceToHost, s),
           "staged send D2H");
      sp[(size_t)i] = sends[i].peer;
      sb[(size_t)i] = hs[(size_t)i].data();
      sz[(size_t)i] = sends[i].bytes;
    }
    for (int i = 0; i < nrecv; ++i) {
      hr[(size_t)i].resize(recvs[i].bytes);
      rp[(size_t)i] = recvs[i].peer;
      rbuf[(size_t)i] = hr[(size_t)i].data();
      rz[(size_t)i] = recvs[i].bytes;
    }
    cuck(cudaStreamSynchronize(s), "staged sendrecv sync");
    if (c->cb_sendrecv(c->cb_ctx, nsend, sp.data(), sb.data(), sz.data(), nrecv, rp.data(), rbuf.data(), rz.data()) != 0)
      throw std::runtime_error("host transport: sendrecv callback failed");
    for (int i = 0; i < nrecv; ++i)
      cuck(cudaMemcpyAsync(recvs[i].ptr, hr[(size_t)i].data(), recvs[i].bytes, cudaMemcpyHostToDevice, s),
           "staged recv H2D");
    cuck(cudaStreamSynchronize(s), "staged sendrecv sync");
    return;
  }
  NcclApi& a = nccl();
  nck(a.GroupStart(), "ncclGroupStart");
  for (int i = 0; i < nsend; ++i)
    nck(a.Send(sends[i].ptr, sends[i].bytes, ncclUint8, sends[i].peer, (ncclComm_t)c->nccl, s), "ncclSend");
  for (int i = 0; i < nrecv; ++i)
    nck(a.Recv(recvs[i].ptr, recvs[i].bytes, ncclUint8, recvs[i].peer, (ncclComm_t)c->nccl, s), "ncclRecv");
  nck(a.GroupEnd(), "ncclGroupEnd");
}

void launch_seg_copy(const double* src, double* dst, const int64_t* src_off, const int64_t* dst_off,
                     const int64_t* len, int nseg, cudaStream_t s) {
  if (nseg <= 0) return;
  seg_copy_kernel<double><<<nseg, 256, 0, s>>>(src, dst, src_off, dst_off, len);
}

void launch_seg_copy_i32(const int32_t* src, int32_t* dst, const int64_t* src_off, const int64_t* dst_off,
                         const int64_t* len, int nseg, cudaStream_t s) {
  if (nseg <= 0) return;
  seg_copy_kernel<int32_t><<<nseg, 128, 0, s>>>(src, dst, src_off, dst_off, len);
}

void launch_rows_gather(const double* src, const int32_t* rows, int64_t nrows, int nrhs, double* dst, cudaStream_t s) {
  if (nrows <= 0) return;
  rows_gather_kernel<<<rows_grid(nrows * nrhs), 256, 0, s>>>(src, rows, nrows, nrhs, dst);
}
void launch_rows_scatter(const double* src, const int32_t* rows, int64_t nrows, int nrhs, double* dst,
                         cudaStream_t s) {
  if (nrows <= 0) return;
  rows_scatter_kernel<<<rows_grid(nrows * nrhs), 256, 0, s>>>(src, rows, nrows, nrhs, dst);
}
void launch_retire_regions(const int32_t* idx, const int64_t* off, const int64_t* len, const int64_t* kid,
                           const int32_t* kout, int nreg, uint8_t* active, cudaStream_t s) {
  if (nreg <= 0) return;
  retire_regions_kernel<<<nreg, 128, 0, s>>>(idx, off, len, kid, kout, active);
}
void launch_rows_zero_unheld(double* v, const uint8_t* holder, int me, int64_t n, int nrhs, cudaStream_t s) {
  if (n <= 0) return;
  rows_zero_unheld_kernel<<<rows_grid(n * nrhs), 256, 0, s>>>(v, holder, me, n, nrhs);
}

}  // namespace hifde

using namespace hifde;

namespace {
thread_local std::string g_comm_err;
}

extern "C" {

const char* hifde_comm_last_error(void) { return g_comm_err.c_str(); }

int hifde_comm_unique_id(uint8_t* id) {
  if (!id) return HIFDE_BADARG;
  NcclApi& a = nccl();
  if (!a.ok) {
    g_comm_err = a.err;
    return HIFDE_CUDA;
  }
  ncclUniqueId u;
  const ncclResult_t r = a.GetUniqueId(&u);
  if (r != ncclSuccess) {
    g_comm_err = std::string("ncclGetUniqueId: ") + a.GetErrorString(r);
    return HIFDE_CUDA;
  }
  static_assert(sizeof(ncclUniqueId) == HIFDE_COMM_ID_BYTES, "NCCL unique id size");
  std::memcpy(id, &u, sizeof u);
  return HIFDE_OK;
}

int hifde_comm_init(const uint8_t* id, int nranks, int rank, int device, hifde_comm_t** out) {
  if (!id || !out || nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks) return HIFDE_BADARG;
  *out = nullptr;
  hifde_comm* c = new hifde_comm;
  c->P = nranks;
  c->rank = rank;
  c->device = device;
  if (nranks > 1) {
    NcclApi& a = nccl();
    if (!a.ok) {
      g_comm_err = a.err;
      delete c;
      return HIFDE_CUDA;
    }
    if (cudaSetDevice(device) != cudaSuccess) {
      g_comm_err = "cudaSetDevice failed";
      delete c;
      return HIFDE_CUDA;
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    ncclComm_t nc = nullptr;
    const ncclResult_t r = a.CommInitRank(&nc, nranks, u, rank);
    if (r != ncclSuccess) {
      g_comm_err = std::string("ncclCommInitRank: ") + a.GetErrorString(r);
      delete c;
      return HIFDE_CUDA;
    }
    c->nccl = nc;
  }
  *out = c;
  return HIFDE_OK;
}

int hifde_comm_emulated(int nranks, int device, hifde_comm_t** out) {
  if (!out || nranks < 1 || nranks > 32) return HIFDE_BADARG;
  hifde_comm* c = new hifde_comm;
  c->P = nranks;
  c->rank = 0;
  c->device = device;
  c->emulated = true;
  *out = c;
  return HIFDE_OK;
}

int hifde_comm_host(int nranks, int rank, int device, hifde_allreduce_cb allreduce, hifde_sendrecv_cb sendrecv,
                    void* ctx, hifde_comm_t** out) {
  if (!out || !allreduce || !sendrecv || nranks < 1 || nranks > 32 || rank < 0 || rank >= nranks) return HIFDE_BADARG;
  hifde_comm* c = new hifde_comm;
  c->P = nranks;
  c->rank = rank;
  c->device = device;
  c->cb_allreduce = allreduce;
  c->cb_sendrecv = sendrecv;
  c->cb_ctx = ctx;
  *out = c;
  return HIFDE_OK;
}

int hifde_comm_info(const hifde_comm_t* c, int* nranks, int* rank, int* emulated) {
  if (!c) return HIFDE_BADARG;
  if (nranks) *nranks = c->P;
  if (rank) *rank = c->rank;
  if (emulated) *emulated = c->emulated ? 1 : 0;
  return HIFDE_OK;
}

void hifde_comm_free(hifde_comm_t* c) {
  if (!c) return;
  if (c->nccl) {
    NcclApi& a = nccl();
    if (a.ok) a.CommDestroy((ncclComm_t)c->nccl);
  }
  delete c;
}

}  // extern "C"
