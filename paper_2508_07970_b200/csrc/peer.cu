// peer.cu — the loss reduction and its cross-rank all-reduce in ONE kernel
// over NVLink peer memory (SURVEY.md §8e collective (1); replaces the
// reference's gather -> coordinator reduce of per-rank sums,
// proj/src/demo.cpp:468-473 / simcore.cpp:304-311, and the separate NCCL
// all-reduce after the loss kernel).
//
// Every rank owns one small device buffer (cudaMalloc, exported with a CUDA
// IPC handle and mapped by every peer of the node):
//   slots[2][kPeerMaxWorld][kPeerMaxFields] fp64   (double-buffered by epoch parity)
//   flags[kPeerMaxWorld] u64                       (flags[q]: last epoch rank q published here)
//   epoch u64, status u32                          (this rank's call counter, timeout flag)
//   gather[2][kPeerMaxWorld][16384] int64          (all-gather banks, by epoch parity)
// One 256-thread block per call: (1) fixed-order reduction of the block
// partials to this rank's sums, (2) stores them into slot [parity][rank] of
// EVERY rank's buffer over NVLink, (3) system fence, then publishes the epoch
// into every rank's flags[rank], (4) waits until all ranks' flags reach the
// epoch, (5) sums the world's slots in rank order — every rank computes the
// identical global result.  A rank can run at most one call ahead of the
// slowest (it needs everyone's flag), so two slot banks suffice.  The epoch
// lives in device memory, so the exchange also works under CUDA-graph replay.
// A wait that exceeds 10 s (%globaltimer) sets status and writes NaN instead
// of hanging; the group is then out of step and should be destroyed.
#include <cuda_runtime.h>

#include <cstring>
#include <new>

#include "common.cuh"

namespace yattb {
namespace {

constexpr int kPeerMaxWorld = YATT_PEER_MAX_WORLD;
constexpr int kPeerMaxFields = 16;
constexpr size_t kSlotBytes = size_t(2) * kPeerMaxWorld * kPeerMaxFields * sizeof(double);
constexpr size_t kFlagOff = kSlotBytes;
constexpr size_t kEpochOff = kFlagOff + kPeerMaxWorld * sizeof(uint64_t);
constexpr size_t kStatusOff = kEpochOff + sizeof(uint64_t);
// all-gather region: gather[2][kPeerMaxWorld][kGatherWords] int64 (parity banks)
constexpr int kGatherWords = YATT_PEER_GATHER_MAX_WORDS;
constexpr size_t kGatherOff = (kStatusOff + 64 + 255) & ~size_t(255);
constexpr size_t kBufBytes = kGatherOff + size_t(2) * kPeerMaxWorld * kGatherWords * 8;

struct PeerArgs {
  uint8_t* buf[kPeerMaxWorld];  // buf[r]: rank r's buffer as mapped in this process
  int32_t world, rank;
};

__device__ __forceinline__ double* slot(uint8_t* b, int parity, int q) {
  return reinterpret_cast<double*>(b) + (size_t(parity) * kPeerMaxWorld + q) * kPeerMaxFields;
}
__device__ __forceinline__ volatile uint64_t* flag(uint8_t* b, int q) {
  return reinterpret_cast<volatile uint64_t*>(b + kFlagOff) + q;
}
__device__ __forceinline__ long long* gather_slot(uint8_t* b, int parity, int q) {
  return reinterpret_cast<long long*>(b + kGatherOff) +
         (size_t(parity) * kPeerMaxWorld + q) * kGatherWords;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread 0: publish this rank's epoch into every rank's flags and wait until
// every rank has published it here (~10 s timeout -> status 1, *fail = 1).
__device__ __forceinline__ void publish_and_wait(const PeerArgs& a, uint64_t epoch, int* fail) {
  uint8_t* mine = a.buf[a.rank];
  __threadfence_system();
  for (int q = 0; q < a.world; ++q) *flag(a.buf[q], a.rank) = epoch;
  const uint64_t t0 = globaltimer_ns();
  for (int q = 0; q < a.world && !*fail; ++q) {
    long long spins = 0;
    while (*flag(mine, q) < epoch) {
      if (spins > 64) __nanosleep(32);  // tight polling first: the usual wait is ~1 us
      // 10 s of wall time: a rank is gone; fail loudly, do not hang
      if ((++spins & 1023) == 0 && globaltimer_ns() - t0 > 10000000000ull) {
        *fail = 1;
        *reinterpret_cast<volatile uint32_t*>(mine + kStatusOff) = 1u;
        break;
      }
    }
  }
  __threadfence_system();
}

// part: nparts records of nf doubles (part[nf*i + f]); out: nf global sums.
__global__ void __launch_bounds__(256) peer_reduce_allreduce_kernel(const double* part,
                                                                     int nparts, int nf,
                                                                     PeerArgs a, double* out) {
  __shared__ double red[kPeerMaxFields][8];
  __shared__ uint64_t s_epoch;
  __shared__ int s_fail;
  double v[kPeerMaxFields];
#pragma unroll
  for (int f = 0; f < kPeerMaxFields; ++f) v[f] = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 256) {
#pragma unroll
    for (int f = 0; f < kPeerMaxFields; ++f)
      if (f < nf) v[f] += part[size_t(nf) * i + f];
  }
  const int w = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < kPeerMaxFields; ++f) {
    if (f >= nf) break;
    v[f] = warp_sum(v[f]);
    if ((threadIdx.x & 31) == 0) red[f][w] = v[f];
  }
  uint8_t* mine = a.buf[a.rank];
  if (threadIdx.x == 0) {
    volatile uint64_t* ep = reinterpret_cast<volatile uint64_t*>(mine + kEpochOff);
    s_epoch = *ep + 1;
    *ep = s_epoch;
    s_fail = 0;
  }
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int parity = int(epoch & 1u);
  // (2) this rank's sums -> slot [parity][rank] of every rank's buffer
  if (threadIdx.x < nf) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += red[threadIdx.x][k];
    for (int q = 0; q < a.world; ++q)
      reinterpret_cast<volatile double*>(slot(a.buf[q], parity, a.rank))[threadIdx.x] = s;
    __threadfence_system();  // each writer orders its slot stores before the flags
  }
  __syncthreads();
  // (3)+(4) publish the epoch (slot stores visible first), wait for everyone's
  if (threadIdx.x == 0) publish_and_wait(a, epoch, &s_fail);
  __syncthreads();
  // (5) identical rank-ordered sum on every rank
  if (threadIdx.x < nf) {
    __threadfence_system();
    double s = 0.0;
    for (int q = 0; q < a.world; ++q)
      s += reinterpret_cast<volatile double*>(slot(mine, parity, q))[threadIdx.x];
    out[threadIdx.x] = s_fail ? __longlong_as_double(0x7ff8000000000000ll) : s;
  }
}

// All-gather + exclusive scan of up to 16 int64 counters per rank in one
// kernel (the dynamic-sampling global offsets): prefix[f] = sum_{q < rank}
// c_q[f], total[f] = sum_q c_q[f] — exact integers, identical on all ranks.
// Shares the slot banks / epoch protocol above (int64 stored as raw words).
__global__ void peer_scan_i64_kernel(const int64_t* in, int nf, PeerArgs a, int64_t* prefix,
                                     int64_t* total) {
  __shared__ uint64_t s_epoch;
  __shared__ int s_fail;
  uint8_t* mine = a.buf[a.rank];
  if (threadIdx.x == 0) {
    volatile uint64_t* ep = reinterpret_cast<volatile uint64_t*>(mine + kEpochOff);
    s_epoch = *ep + 1;
    *ep = s_epoch;
    s_fail = 0;
  }
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int parity = int(epoch & 1u);
  if (threadIdx.x < nf) {
    const long long v = in[threadIdx.x];
    for (int q = 0; q < a.world; ++q)
      reinterpret_cast<volatile long long*>(slot(a.buf[q], parity, a.rank))[threadIdx.x] = v;
    __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x == 0) publish_and_wait(a, epoch, &s_fail);
  __syncthreads();
  if (threadIdx.x < nf) {
    __threadfence_system();
    long long pre = 0, tot = 0;
    for (int q = 0; q < a.world; ++q) {
      const long long c = reinterpret_cast<volatile long long*>(slot(mine, parity, q))[threadIdx.x];
      if (q < a.rank) pre += c;
      tot += c;
    }
    if (prefix) prefix[threadIdx.x] = s_fail ? -1 : pre;
    if (total) total[threadIdx.x] = s_fail ? -1 : tot;
  }
}

// All-gather of n int64 words per rank (rank-major out[world * n]): the
// binary round-report / microbatch exchange of the dynamic-sampling loop
// (replaces the reference's JSON submit_round RPC, demo.cpp:32-76, and the
// NCCL all-gather).  Each rank pushes its words into gather[parity][rank] of
// every rank's buffer over NVLink, fences, publishes the epoch; then copies
// the world's words from its own buffer.  Same epoch / parity protocol as
// the kernels above; on timeout every output word is -1.
__global__ void __launch_bounds__(256) peer_allgather_i64_kernel(const int64_t* in, int n,
                                                                  PeerArgs a, int64_t* out) {
  __shared__ uint64_t s_epoch;
  __shared__ int s_fail;
  uint8_t* mine = a.buf[a.rank];
  if (threadIdx.x == 0) {
    volatile uint64_t* ep = reinterpret_cast<volatile uint64_t*>(mine + kEpochOff);
    s_epoch = *ep + 1;
    *ep = s_epoch;
    s_fail = 0;
  }
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int parity = int(epoch & 1u);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const long long v = in[i];
    for (int q = 0; q < a.world; ++q)
      reinterpret_cast<volatile long long*>(gather_slot(a.buf[q], parity, a.rank))[i] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) publish_and_wait(a, epoch, &s_fail);
  __syncthreads();
  __threadfence_system();
  for (int q = 0; q < a.world; ++q) {
    const volatile long long* src = gather_slot(mine, parity, q);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      out[size_t(q) * n + i] = s_fail ? -1 : src[i];
  }
}

}  // namespace

int peer_reduce_launch(const PeerArgs& a, const double* part, int nparts, int nf, double* out,
                       cudaStream_t st) {
  peer_reduce_allreduce_kernel<<<1, 256, 0, st>>>(part, nparts, nf, a, out);
  return check_launch("peer_reduce_allreduce_kernel");
}

// loss.cu: block partials of the policy loss (no final reduce).
int policy_loss_parts_launch(const float* logp, const float* old_logp, const float* adv,
                             const float* kl, const float* ent, const uint8_t* mask, int64_t n,
                             const int64_t* cu, int64_t nseq, const yatt_loss_config* cfg,
                             void* ws, size_t ws_bytes, int* nparts, cudaStream_t st);

}  // namespace yattb

struct yatt_peer {
  int32_t world, rank;
  uint8_t* local;
  uint8_t* mapped[YATT_PEER_MAX_WORLD];
  bool opened[YATT_PEER_MAX_WORLD];
  bool connected;
};

using namespace yattb;

extern "C" {

int yatt_peer_create(int32_t world, int32_t rank, yatt_peer_t* out, uint8_t* h_handle) {
  static_assert(sizeof(cudaIpcMemHandle_t) == YATT_PEER_HANDLE_BYTES, "IPC handle size");
  YATT_REQUIRE(world >= 1 && world <= kPeerMaxWorld, YATT_ERR_CONFIG,
               "peer_create: world must be in [1, %d]", kPeerMaxWorld);
  YATT_REQUIRE(rank >= 0 && rank < world, YATT_ERR_RANK, "peer_create: rank out of range");
  YATT_REQUIRE(out != nullptr && h_handle != nullptr, YATT_ERR_CONFIG, "peer_create: null arg");
  yatt_peer* p = new (std::nothrow) yatt_peer{};
  YATT_REQUIRE(p != nullptr, YATT_ERR_CONFIG, "peer_create: out of host memory");
  p->world = world;
  p->rank = rank;
  cudaError_t e = cudaMalloc(&p->local, kBufBytes);
  if (e == cudaSuccess) e = cudaMemset(p->local, 0, kBufBytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p->local);
  if (e != cudaSuccess) {
    if (p->local) cudaFree(p->local);
    delete p;
    return set_error(YATT_ERR_CUDA, "peer_create: %s", cudaGetErrorString(e));
  }
  std::memcpy(h_handle, &h, sizeof(h));
  p->mapped[rank] = p->local;
  *out = p;
  return YATT_OK;
}

int yatt_peer_connect(yatt_peer_t p, const uint8_t* h_handles) {
  YATT_REQUIRE(p != nullptr && h_handles != nullptr, YATT_ERR_CONFIG, "peer_connect: null arg");
  for (int q = 0; q < p->world; ++q) {
    if (q == p->rank || p->opened[q]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, h_handles + size_t(q) * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    YATT_TRY_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->mapped[q] = static_cast<uint8_t*>(ptr);
    p->opened[q] = true;
  }
  YATT_TRY_CUDA(cudaDeviceSynchronize());
  p->connected = true;
  return YATT_OK;
}

int yatt_peer_destroy(yatt_peer_t p) {
  if (p == nullptr) return YATT_OK;
  for (int q = 0; q < p->world; ++q)
    if (p->opened[q]) cudaIpcCloseMemHandle(p->mapped[q]);
  if (p->local) cudaFree(p->local);
  delete p;
  return YATT_OK;
}

int yatt_peer_world(yatt_peer_t p, int32_t* world, int32_t* rank) {
  YATT_REQUIRE(p != nullptr && world != nullptr && rank != nullptr, YATT_ERR_CONFIG,
               "peer_world: null arg");
  YATT_REQUIRE(p->connected, YATT_ERR_CONFIG, "peer: create + connect the peer group first");
  *world = p->world;
  *rank = p->rank;
  return YATT_OK;
}

int yatt_peer_status(yatt_peer_t p, int32_t* h_status) {
  YATT_REQUIRE(p != nullptr && h_status != nullptr, YATT_ERR_CONFIG, "peer_status: null arg");
  uint32_t s = 0;
  YATT_TRY_CUDA(cudaMemcpy(&s, p->local + kStatusOff, sizeof(s), cudaMemcpyDeviceToHost));
  *h_status = int32_t(s);
  return YATT_OK;
}

static int peer_args(yatt_peer_t p, PeerArgs* a) {
  YATT_REQUIRE(p != nullptr && p->connected, YATT_ERR_CONFIG,
               "peer: create + connect the peer group first");
  *a = PeerArgs{};
  for (int q = 0; q < p->world; ++q) a->buf[q] = p->mapped[q];
  a->world = p->world;
  a->rank = p->rank;
  return YATT_OK;
}

int yatt_peer_allreduce_f64(yatt_peer_t p, const double* d_in, int32_t n, double* d_out,
                            void* stream) {
  YATT_REQUIRE(n >= 1 && n <= kPeerMaxFields, YATT_ERR_CONFIG,
               "peer_allreduce_f64: n must be in [1, %d]", kPeerMaxFields);
  YATT_REQUIRE(d_in && d_out, YATT_ERR_CONFIG, "peer_allreduce_f64: null pointer");
  PeerArgs a;
  const int rc = peer_args(p, &a);
  if (rc) return rc;
  return peer_reduce_launch(a, d_in, 1, n, d_out, as_stream(stream));
}

int yatt_peer_scan_i64(yatt_peer_t p, const int64_t* d_in, int32_t n, int64_t* d_prefix,
                       int64_t* d_total, void* stream) {
  YATT_REQUIRE(n >= 1 && n <= kPeerMaxFields, YATT_ERR_CONFIG,
               "peer_scan_i64: n must be in [1, %d]", kPeerMaxFields);
  YATT_REQUIRE(d_in != nullptr, YATT_ERR_CONFIG, "peer_scan_i64: null input");
  PeerArgs a;
  const int rc = peer_args(p, &a);
  if (rc) return rc;
  peer_scan_i64_kernel<<<1, 32, 0, as_stream(stream)>>>(d_in, n, a, d_prefix, d_total);
  return check_launch("peer_scan_i64_kernel");
}

int yatt_peer_allgather_i64(yatt_peer_t p, const int64_t* d_in, int32_t n, int64_t* d_out,
                            void* stream) {
  YATT_REQUIRE(n >= 1 && n <= kGatherWords, YATT_ERR_CONFIG,
               "peer_allgather_i64: n must be in [1, %d]", kGatherWords);
  YATT_REQUIRE(d_in && d_out, YATT_ERR_CONFIG, "peer_allgather_i64: null pointer");
  PeerArgs a;
  const int rc = peer_args(p, &a);
  if (rc) return rc;
  peer_allgather_i64_kernel<<<1, 256, 0, as_stream(stream)>>>(d_in, n, a, d_out);
  return check_launch("peer_allgather_i64_kernel");
}

int yatt_policy_loss_allreduce(yatt_peer_t p, const float* logp, const float* old_logp,
                               const float* adv, const float* kl, const float* ent,
                               const uint8_t* mask, int64_t n, const int64_t* cu, int64_t nseq,
                               const yatt_loss_config* cfg, yatt_loss_sums* d_sums, void* ws,
                               size_t ws_bytes, void* stream) {
  YATT_REQUIRE(d_sums != nullptr, YATT_ERR_CONFIG, "policy_loss_allreduce: null sums");
  PeerArgs a;
  int rc = peer_args(p, &a);
  if (rc) return rc;
  int nparts = 0;
  rc = policy_loss_parts_launch(logp, old_logp, adv, kl, ent, mask, n, cu, nseq, cfg, ws, ws_bytes,
                                &nparts, as_stream(stream));
  if (rc) return rc;
  return peer_reduce_launch(a, static_cast<const double*>(ws), nparts, 8,
                            reinterpret_cast<double*>(d_sums), as_stream(stream));
}

}  // extern "C"
