// comm.cu — cross-rank collectives for the parallel-controller ranks.
//
// Replaces the reference's gather -> coordinator reduce -> broadcast of
// ShardRoundReports over JSON/TCP RPC (proj/src/demo.cpp:32-76, :261-274,
// :336-339; reduce at proj/src/simcore.cpp:304-311) with NCCL collectives on
// device buffers over NVLink/NVSwitch.  Messages are tiny (tens of bytes):
//   * all-reduce (sum) of the loss sums / token count  (fp64)
//   * all-reduce (sum) of integer round counters        (int64)
//   * all-gather of per-rank survivor counts            (int64) -> offsets
// The unique id travels out of band (torch.distributed store, or the
// reference's own RPC rendezvous, demo.cpp:409-428).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <new>

#include "common.cuh"

struct yatt_comm {
  ncclComm_t comm;
  int32_t nranks;
  int32_t rank;
};

#define YATT_TRY_NCCL(expr)                                                            \
  do {                                                                                 \
    ncclResult_t _r = (expr);                                                          \
    if (_r != ncclSuccess)                                                             \
      return ::yattb::set_error(YATT_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(_r)); \
  } while (0)

using namespace yattb;

extern "C" {

int yatt_comm_unique_id(uint8_t* h_id) {
  static_assert(sizeof(ncclUniqueId) == YATT_COMM_ID_BYTES, "ncclUniqueId size");
  YATT_REQUIRE(h_id != nullptr, YATT_ERR_CONFIG, "comm_unique_id: null output");
  ncclUniqueId id;
  YATT_TRY_NCCL(ncclGetUniqueId(&id));
  std::memcpy(h_id, &id, sizeof(id));
  return YATT_OK;
}

int yatt_comm_init(int32_t nranks, int32_t rank, const uint8_t* h_id, yatt_comm_t* out) {
  YATT_REQUIRE(nranks > 0, YATT_ERR_CONFIG, "comm_init: nranks must be positive");
  YATT_REQUIRE(rank >= 0 && rank < nranks, YATT_ERR_RANK, "comm_init: rank out of range");
  YATT_REQUIRE(h_id != nullptr && out != nullptr, YATT_ERR_CONFIG, "comm_init: null argument");
  ncclUniqueId id;
  std::memcpy(&id, h_id, sizeof(id));
  yatt_comm* c = new (std::nothrow) yatt_comm{nullptr, nranks, rank};
  YATT_REQUIRE(c != nullptr, YATT_ERR_CONFIG, "comm_init: out of host memory");
  const ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_error(YATT_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return YATT_OK;
}

int yatt_comm_destroy(yatt_comm_t c) {
  if (c == nullptr) return YATT_OK;
  const ncclResult_t r = ncclCommDestroy(c->comm);
  delete c;
  YATT_REQUIRE(r == ncclSuccess, YATT_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return YATT_OK;
}

int yatt_comm_allreduce_f64(yatt_comm_t c, double* buf, int64_t count, void* stream) {
  YATT_REQUIRE(c != nullptr && count >= 0, YATT_ERR_CONFIG, "allreduce_f64: bad arguments");
  YATT_TRY_NCCL(ncclAllReduce(buf, buf, size_t(count), ncclFloat64, ncclSum, c->comm,
                              as_stream(stream)));
  return YATT_OK;
}

int yatt_comm_allreduce_i64(yatt_comm_t c, int64_t* buf, int64_t count, void* stream) {
  YATT_REQUIRE(c != nullptr && count >= 0, YATT_ERR_CONFIG, "allreduce_i64: bad arguments");
  YATT_TRY_NCCL(ncclAllReduce(buf, buf, size_t(count), ncclInt64, ncclSum, c->comm,
                              as_stream(stream)));
  return YATT_OK;
}

int yatt_comm_allgather_i64(yatt_comm_t c, const int64_t* send, int64_t* recv, int64_t count,
                            void* stream) {
  YATT_REQUIRE(c != nullptr && count >= 0, YATT_ERR_CONFIG, "allgather_i64: bad arguments");
  YATT_TRY_NCCL(ncclAllGather(send, recv, size_t(count), ncclInt64, c->comm, as_stream(stream)));
  return YATT_OK;
}

}  // extern "C"
