// Exchange primitives of the sharded engine (include/qsv.h "sharding").
//
// A remap step of dist.py trades, for every rank pair (r, p), the slice
// {x : bits ls of x == d_r} of shard r with the slice {x : bits ls == d_p}
// of shard p.  With peer memory (same process: another shard's pointer;
// another process: a CUDA IPC mapping) that trade is one in-place kernel
// over NVLink: each element is loaded from both sides and stored crosswise,
// so one HBM read + write on each side plus the NVLink read + write -- no
// staging buffer, no pack / unpack copies, no NCCL kernel.  Both owners of a
// pair run it at once on disjoint halves of the slice, so both GPUs' SMs and
// both NVLink directions carry the exchange.
//
// Ordering against the peer's own work is the caller's (dist.py: a device
// barrier before and after an exchange step); within the step different
// pairs touch disjoint slices, so the 2^k - 1 rounds need no barrier between
// them.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "qsv_internal.cuh"

namespace qsv {
namespace {

struct SliceMap {
  int k;
  int pos[QSV_MAX_SLICE_BITS];  // ascending bit positions
  uint64_t va, vb;              // the fixed bits of the two slices
};

constexpr int kSwapThreads = 256;
constexpr int kSwapFatThreads = 1024;  // SM-limited launches: one fat CTA per SM
constexpr int kSwapPer = 4;  // elements per thread in flight (loads before stores)

__device__ __forceinline__ uint64_t spread(uint64_t j, const SliceMap& m) {
#pragma unroll 1
  for (int i = 0; i < m.k; ++i) {
    const int p = m.pos[i];
    j = ((j >> p) << (p + 1)) | (j & ((1ULL << p) - 1));
  }
  return j;
}

template <int Threads>
__global__ void __launch_bounds__(Threads) k_slice_swap(double2* __restrict__ a,
                                                        double2* __restrict__ b, SliceMap m,
                                                        uint64_t j0, uint64_t j1) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = j0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < j1;
       base += stride * kSwapPer) {
    uint64_t ia[kSwapPer], ib[kSwapPer];
    double2 va[kSwapPer], vb[kSwapPer];
#pragma unroll
    for (int i = 0; i < kSwapPer; ++i) {
      const uint64_t j = base + i * stride;
      const uint64_t x = spread(j, m);
      ia[i] = x | m.va;
      ib[i] = x | m.vb;
      if (j < j1) {
        va[i] = a[ia[i]];
        vb[i] = b[ib[i]];
      }
    }
#pragma unroll
    for (int i = 0; i < kSwapPer; ++i) {
      if (base + i * stride < j1) {
        a[ia[i]] = vb[i];
        b[ib[i]] = va[i];
      }
    }
  }
}

// 32-byte variant: when the lowest slice bit is above bit 0, slice elements
// 2i and 2i + 1 are adjacent amplitudes, so a thread moves the pair with one
// 256-bit load / store on each side (half the memory instructions per byte,
// the form of the HBM-bound gate kernels); pair range [p0, p1)
template <int Threads>
__global__ void __launch_bounds__(Threads) k_slice_swap2(double2* __restrict__ a,
                                                         double2* __restrict__ b, SliceMap m,
                                                         uint64_t p0, uint64_t p1) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = p0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; base < p1;
       base += stride * kSwapPer) {
    uint64_t ia[kSwapPer], ib[kSwapPer];
    Amp2 va[kSwapPer], vb[kSwapPer];
#pragma unroll
    for (int i = 0; i < kSwapPer; ++i) {
      const uint64_t j = base + i * stride;
      const uint64_t x = spread(j << 1, m);
      ia[i] = x | m.va;
      ib[i] = x | m.vb;
      if (j < p1) {
        va[i] = ld2(a + ia[i]);
        vb[i] = ld2(b + ib[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < kSwapPer; ++i) {
      if (base + i * stride < p1) {
        st2(a + ia[i], vb[i]);
        st2(b + ib[i], va[i]);
      }
    }
  }
}

// QSV_SWAP_VEC=0 forces the 16-byte kernel (A/B of the exchange step)
bool swap_vec2_enabled() {
  static const int on = [] {
    const char* e = getenv("QSV_SWAP_VEC");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

}  // namespace
}  // namespace qsv

using namespace qsv;

extern "C" {

int qsv_ipc_export(const qsv_state* st, void* handle_out) {
  if (!st || !handle_out) {
    set_error("null state or handle buffer");
    return QSV_EINVAL;
  }
  if (st->view) {
    set_error("a state view cannot be exported (export the state that owns the buffer)");
    return QSV_EINVAL;
  }
  if (!st->plain && st->dim * sizeof(double2) <= (1ULL << 30)) {
    set_error("state was not created with qsv_state_create_shared (pooled memory cannot be "
              "exported)");
    return QSV_EINVAL;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == QSV_IPC_HANDLE_BYTES, "IPC handle size");
  DeviceGuard dg(st->device);
  cudaIpcMemHandle_t h;
  QSV_TRY(cudaIpcGetMemHandle(&h, st->amps));
  std::memcpy(handle_out, &h, sizeof(h));
  return QSV_OK;
}

int qsv_ipc_open(const void* handle, int device, void** peer_amps) {
  if (!handle || !peer_amps) {
    set_error("null handle or output pointer");
    return QSV_EINVAL;
  }
  DeviceGuard dg(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  QSV_TRY(cudaIpcOpenMemHandle(peer_amps, h, cudaIpcMemLazyEnablePeerAccess));
  return QSV_OK;
}

int qsv_ipc_close(int device, void* peer_amps) {
  if (!peer_amps) return QSV_OK;
  DeviceGuard dg(device);
  QSV_TRY(cudaIpcCloseMemHandle(peer_amps));
  return QSV_OK;
}

int qsv_slice_swap(qsv_state* st, void* peer_amps, const int* ls, int k, uint64_t d_mine,
                   uint64_t d_peer, uint64_t j0, uint64_t j1) {
  if (!st || !peer_amps || (k > 0 && !ls)) {
    set_error("null state, peer buffer or slice bits");
    return QSV_EINVAL;
  }
  if (k < 0 || k > QSV_MAX_SLICE_BITS || k > st->n) {
    set_error("slice bit count %d out of range", k);
    return QSV_EINVAL;
  }
  SliceMap m{};
  m.k = k;
  uint64_t seen = 0;
  for (int i = 0; i < k; ++i) {
    if (ls[i] < 0 || ls[i] >= st->n || ((seen >> ls[i]) & 1)) {
      set_error("slice bit %d invalid or repeated", ls[i]);
      return QSV_EINVAL;
    }
    seen |= 1ULL << ls[i];
    m.pos[i] = ls[i];
    m.va |= ((d_mine >> i) & 1ULL) << ls[i];
    m.vb |= ((d_peer >> i) & 1ULL) << ls[i];
  }
  std::sort(m.pos, m.pos + k);
  const uint64_t count = st->dim >> k;
  if (j0 > j1 || j1 > count) {
    set_error("slice range [%llu, %llu) outside [0, %llu)", (unsigned long long)j0,
              (unsigned long long)j1, (unsigned long long)count);
    return QSV_EINVAL;
  }
  if (j0 == j1) return QSV_OK;
  DeviceGuard dg(st->device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st->device);
  double2* peer = static_cast<double2*>(peer_amps);
  const bool vec2 = swap_vec2_enabled() && (k == 0 || m.pos[0] >= 1) && !(j0 & 1) && !(j1 & 1) &&
                    !(reinterpret_cast<uintptr_t>(peer) & 31) &&
                    !(reinterpret_cast<uintptr_t>(st->amps) & 31);
  if (vec2) {
    const uint64_t q0 = j0 >> 1, q1 = j1 >> 1;
    const int threads = st->sm_limit > 0 ? kSwapFatThreads : kSwapThreads;
    const uint64_t per_block = (uint64_t)threads * kSwapPer;
    const uint64_t want = (q1 - q0 + per_block - 1) / per_block;
    const uint64_t cap = st->sm_limit > 0 ? (uint64_t)std::min(st->sm_limit, sms) : (uint64_t)sms * 8;
    const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, cap));
    if (st->sm_limit > 0)
      k_slice_swap2<kSwapFatThreads><<<blocks, kSwapFatThreads, 0, st->stream>>>(st->amps, peer, m,
                                                                                  q0, q1);
    else
      k_slice_swap2<kSwapThreads><<<blocks, kSwapThreads, 0, st->stream>>>(st->amps, peer, m, q0,
                                                                          q1);
    QSV_TRY(cudaGetLastError());
    return QSV_OK;
  }
  if (st->sm_limit > 0) {
    // overlapped with tile passes on another stream: at most sm_limit SMs,
    // one 1024-thread CTA each (the tile kernel's CTAs fill a whole SM, so
    // thin CTAs spread over many SMs would block its launch)
    const uint64_t per_block = (uint64_t)kSwapFatThreads * kSwapPer;
    const uint64_t want = (j1 - j0 + per_block - 1) / per_block;
    const int blocks = (int)std::min<uint64_t>(want, (uint64_t)std::min(st->sm_limit, sms));
    k_slice_swap<kSwapFatThreads><<<blocks, kSwapFatThreads, 0, st->stream>>>(
        st->amps, peer, m, j0, j1);
  } else {
    const uint64_t per_block = (uint64_t)kSwapThreads * kSwapPer;
    const uint64_t want = (j1 - j0 + per_block - 1) / per_block;
    const int blocks = (int)std::min<uint64_t>(want, (uint64_t)sms * 8);
    k_slice_swap<kSwapThreads><<<blocks, kSwapThreads, 0, st->stream>>>(
        st->amps, peer, m, j0, j1);
  }
  QSV_TRY(cudaGetLastError());
  return QSV_OK;
}

}  // extern "C"
