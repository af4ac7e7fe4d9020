// NCCL communicator of the sharded engine, inside libqsv (include/qsv.h
// "communicator").
//
// dist.py needs three collective services between the processes that hold
// shards: a device-side barrier that orders every rank's queued shard work
// (before and after a peer-memory exchange step), a sum over ranks of a few
// doubles (norms, expectation values), and -- where shards cannot be mapped
// into each other's address space -- the slice exchange of a remap step as
// point-to-point transfers.  All three run here on the shard's own CUDA
// stream through NCCL's C API; torch.distributed is used only to hand the
// 128-byte NCCL unique id from rank 0 to the others (rendezvous).
//
// NCCL is loaded on first use with dlopen("libnccl.so.2"), so libqsv does not
// depend on it for single-GPU work, and a process that already loaded NCCL
// (torch's copy) reuses that library instead of mapping a second one.
//
// Slice exchange: the slice {x : bits ls of x == d} of a shard is gathered
// into a staging buffer by one kernel (strided reads, contiguous writes),
// sent with ncclSend while the partner's slice arrives with ncclRecv in the
// same group, and scattered back into the slice {x : bits ls == d_recv}
// (chunked so staging stays bounded).  Reference: none (the reference is
// single-process); this is the "NCCL send/recv" exchange of the
// north star, the fallback of the in-place NVLink kernel (qsv_exchange.cu).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "qsv_internal.cuh"

namespace qsv {
namespace {

struct NcclApi {
  bool loaded = false;
  std::string error;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  decltype(&ncclGetVersion) getVersion = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define QSV_NCCL_SYM(field, sym)                                      \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #sym)); \
  if (!api.field) {                                                   \
    api.error = "libnccl.so.2 lacks " #sym;                           \
    return;                                                           \
  }
    QSV_NCCL_SYM(getUniqueId, ncclGetUniqueId);
    QSV_NCCL_SYM(commInitRank, ncclCommInitRank);
    QSV_NCCL_SYM(commDestroy, ncclCommDestroy);
    QSV_NCCL_SYM(allReduce, ncclAllReduce);
    QSV_NCCL_SYM(send, ncclSend);
    QSV_NCCL_SYM(recv, ncclRecv);
    QSV_NCCL_SYM(groupStart, ncclGroupStart);
    QSV_NCCL_SYM(groupEnd, ncclGroupEnd);
    QSV_NCCL_SYM(errorString, ncclGetErrorString);
    QSV_NCCL_SYM(getVersion, ncclGetVersion);
#undef QSV_NCCL_SYM
    api.loaded = true;
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  set_error("%s: %s", what, nccl().errorString ? nccl().errorString(r) : "NCCL error");
  return QSV_ECUDA;
}

#define QSV_NCCL(call, what)                                  \
  do {                                                        \
    const ncclResult_t r__ = (call);                          \
    if (r__ != ncclSuccess) return nccl_fail(r__, what);      \
  } while (0)

int need_nccl() {
  if (!nccl().loaded) {
    set_error("%s", nccl().error.c_str());
    return QSV_EUNSUPPORTED;
  }
  return QSV_OK;
}

// slice element j (0 <= j < 2^(n-k)) -> amplitude index: zero bits inserted
// at the ascending slice positions, then the slice's fixed bits OR-ed in
struct SliceBits {
  int k;
  int pos[QSV_MAX_SLICE_BITS];
  uint64_t value;
};

__device__ __forceinline__ uint64_t slice_index(uint64_t j, const SliceBits& m) {
#pragma unroll 1
  for (int i = 0; i < m.k; ++i) {
    const int p = m.pos[i];
    j = ((j >> p) << (p + 1)) | (j & ((1ULL << p) - 1));
  }
  return j | m.value;
}

constexpr int kPackThreads = 256;
constexpr int kPackPer = 4;

// out[j - j0] = a[slice(j)] (gather) or a[slice(j)] = in[j - j0] (scatter)
template <bool Gather>
__global__ void __launch_bounds__(kPackThreads)
    k_slice_pack(double2* __restrict__ a, double2* __restrict__ buf, SliceBits m, uint64_t j0,
                 uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < count;
       base += stride * kPackPer) {
    double2 v[kPackPer];
    uint64_t idx[kPackPer];
#pragma unroll
    for (int i = 0; i < kPackPer; ++i) {
      const uint64_t j = base + i * stride;
      idx[i] = slice_index(j0 + j, m);
      if (j < count) v[i] = Gather ? a[idx[i]] : buf[j];
    }
#pragma unroll
    for (int i = 0; i < kPackPer; ++i) {
      const uint64_t j = base + i * stride;
      if (j < count) {
        if (Gather) buf[j] = v[i];
        else a[idx[i]] = v[i];
      }
    }
  }
}

int launch_pack(bool gather, double2* a, double2* buf, const SliceBits& m, uint64_t j0,
                uint64_t count, int device, cudaStream_t s) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const uint64_t per_block = (uint64_t)kPackThreads * kPackPer;
  const int blocks = (int)std::max<uint64_t>(
      1, std::min<uint64_t>((count + per_block - 1) / per_block, (uint64_t)sms * 8));
  if (gather) k_slice_pack<true><<<blocks, kPackThreads, 0, s>>>(a, buf, m, j0, count);
  else k_slice_pack<false><<<blocks, kPackThreads, 0, s>>>(a, buf, m, j0, count);
  QSV_TRY(cudaGetLastError());
  return QSV_OK;
}

int make_slice(const qsv_state* st, const int* ls, int k, uint64_t d, SliceBits& m) {
  if (k < 0 || k > QSV_MAX_SLICE_BITS || k > st->n || (k > 0 && !ls)) {
    set_error("slice bit count %d out of range", k);
    return QSV_EINVAL;
  }
  m.k = k;
  m.value = 0;
  uint64_t seen = 0;
  for (int i = 0; i < k; ++i) {
    if (ls[i] < 0 || ls[i] >= st->n || ((seen >> ls[i]) & 1ULL)) {
      set_error("slice bit %d invalid or repeated", ls[i]);
      return QSV_EINVAL;
    }
    seen |= 1ULL << ls[i];
    m.pos[i] = ls[i];
    m.value |= ((d >> i) & 1ULL) << ls[i];
  }
  std::sort(m.pos, m.pos + k);
  return QSV_OK;
}

}  // namespace
}  // namespace qsv

struct qsv_comm {
  ncclComm_t comm = nullptr;
  int device = 0;
  int nranks = 1, rank = 0;
  double* scalars = nullptr;       // allreduce scratch (device)
  double2* stage = nullptr;        // send half | recv half
  size_t stage_elems = 0;          // elements per half
  cudaStream_t stage_stream = nullptr;  // stream the staging was last used on
};

using namespace qsv;

extern "C" {

int qsv_comm_available(void) { return nccl().loaded ? 1 : 0; }

int qsv_comm_unique_id(void* id_out) {
  if (!id_out) {
    set_error("null id buffer");
    return QSV_EINVAL;
  }
  static_assert(sizeof(ncclUniqueId) == QSV_COMM_ID_BYTES, "NCCL unique id size");
  int rc = need_nccl();
  if (rc) return rc;
  ncclUniqueId id;
  QSV_NCCL(nccl().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  return QSV_OK;
}

int qsv_comm_create(const void* id, int nranks, int rank, int device, qsv_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("bad communicator arguments (nranks %d, rank %d)", nranks, rank);
    return QSV_EINVAL;
  }
  *out = nullptr;
  int rc = need_nccl();
  if (rc) return rc;
  DeviceGuard dg(device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  qsv_comm* c = new qsv_comm();
  c->device = device;
  c->nranks = nranks;
  c->rank = rank;
  const ncclResult_t r = nccl().commInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  cudaError_t e = cudaMalloc(&c->scalars, 64 * sizeof(double));
  if (e != cudaSuccess) {
    nccl().commDestroy(c->comm);
    delete c;
    return cuda_fail(e, "cudaMalloc(communicator scratch)");
  }
  *out = c;
  return QSV_OK;
}

int qsv_comm_destroy(qsv_comm* c) {
  if (!c) return QSV_OK;
  DeviceGuard dg(c->device);
  cudaDeviceSynchronize();
  if (c->comm) nccl().commDestroy(c->comm);
  if (c->scalars) cudaFree(c->scalars);
  if (c->stage) cudaFree(c->stage);
  delete c;
  return QSV_OK;
}

int qsv_comm_rank(const qsv_comm* c, int* rank, int* nranks) {
  if (!c || !rank || !nranks) return QSV_EINVAL;
  *rank = c->rank;
  *nranks = c->nranks;
  return QSV_OK;
}

int qsv_comm_barrier(qsv_comm* c, qsv_state* st) {
  if (!c || !st) {
    set_error("null communicator or state");
    return QSV_EINVAL;
  }
  DeviceGuard dg(c->device);
  // one-element sum on the shard stream: it completes on every rank only
  // after all ranks' earlier work on their shard streams -- no host wait
  QSV_NCCL(nccl().allReduce(c->scalars, c->scalars, 1, ncclFloat64, ncclSum, c->comm, st->stream),
           "ncclAllReduce(barrier)");
  return QSV_OK;
}

int qsv_comm_allreduce_sum(qsv_comm* c, qsv_state* st, double* values, int count) {
  if (!c || !st || !values || count < 0 || count > 64) {
    set_error("bad allreduce arguments (count %d, at most 64)", count);
    return QSV_EINVAL;
  }
  if (count == 0) return QSV_OK;
  DeviceGuard dg(c->device);
  QSV_TRY(cudaMemcpyAsync(c->scalars, values, count * sizeof(double), cudaMemcpyHostToDevice,
                          st->stream));
  QSV_NCCL(nccl().allReduce(c->scalars, c->scalars, count, ncclFloat64, ncclSum, c->comm,
                            st->stream),
           "ncclAllReduce");
  QSV_TRY(cudaMemcpyAsync(values, c->scalars, count * sizeof(double), cudaMemcpyDeviceToHost,
                          st->stream));
  QSV_TRY(cudaStreamSynchronize(st->stream));
  return QSV_OK;
}

int qsv_comm_slice_exchange(qsv_comm* c, qsv_state* st, int peer, const int* ls, int k,
                            uint64_t d_send, uint64_t d_recv, uint64_t chunk_bytes) {
  if (!c || !st) {
    set_error("null communicator or state");
    return QSV_EINVAL;
  }
  if (peer < 0 || peer >= c->nranks) {
    set_error("peer rank %d outside [0, %d)", peer, c->nranks);
    return QSV_EINVAL;
  }
  SliceBits ms{}, mr{};
  int rc = make_slice(st, ls, k, d_send, ms);
  if (!rc) rc = make_slice(st, ls, k, d_recv, mr);
  if (rc) return rc;
  DeviceGuard dg(c->device);
  const uint64_t count = st->dim >> k;
  const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(count, (chunk_bytes ? chunk_bytes
                                                                                      : (1ULL << 30)) /
                                                                             sizeof(double2)));
  if (c->stage_elems < chunk) {
    if (c->stage) {
      QSV_TRY(cudaStreamSynchronize(c->stage_stream ? c->stage_stream : st->stream));
      QSV_TRY(cudaFree(c->stage));
      c->stage = nullptr;
    }
    QSV_TRY(cudaMalloc(&c->stage, 2 * chunk * sizeof(double2)));
    c->stage_elems = chunk;
  }
  if (c->stage_stream && c->stage_stream != st->stream) {
    // the staging buffer may still be read by the last exchange's stream
    cudaEvent_t ev;
    QSV_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    QSV_TRY(cudaEventRecord(ev, c->stage_stream));
    QSV_TRY(cudaStreamWaitEvent(st->stream, ev, 0));
    cudaEventDestroy(ev);
  }
  c->stage_stream = st->stream;
  double2* sendb = c->stage;
  double2* recvb = c->stage + c->stage_elems;
  for (uint64_t j0 = 0; j0 < count; j0 += chunk) {
    const uint64_t m = std::min(chunk, count - j0);
    rc = launch_pack(true, st->amps, sendb, ms, j0, m, c->device, st->stream);
    if (rc) return rc;
    QSV_NCCL(nccl().groupStart(), "ncclGroupStart");
    QSV_NCCL(nccl().send(sendb, 2 * m, ncclFloat64, peer, c->comm, st->stream), "ncclSend");
    QSV_NCCL(nccl().recv(recvb, 2 * m, ncclFloat64, peer, c->comm, st->stream), "ncclRecv");
    QSV_NCCL(nccl().groupEnd(), "ncclGroupEnd");
    rc = launch_pack(false, st->amps, recvb, mr, j0, m, c->device, st->stream);
    if (rc) return rc;
  }
  return QSV_OK;
}

}  // extern "C"
