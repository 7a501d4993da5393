// NCCL communicator of the multi-GPU build: the collectives of the subtree-
// sharded build -- all-reduce of the world cube and of the counting grids, the all-to-all
// point exchange, the gather of subtree-root voxels to rank 0 -- issued by the library on the
// build's stream over NVLink / NVSwitch.  NCCL is loaded at first use (dlopen "libnccl.so.2":
// the copy torch already loaded, else the system one), so the library itself has no link-time
// NCCL dependency and single-GPU users never touch it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "kernels.h"

namespace lod {
int fail(int code, const char* fmt, ...);
}

using namespace lod;

namespace {

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SYM(f) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, "nccl" #f))
    SYM(GetUniqueId);
    SYM(CommInitRank);
    SYM(CommDestroy);
    SYM(AllReduce);
    SYM(AllGather);
    SYM(Send);
    SYM(Recv);
    SYM(GroupStart);
    SYM(GroupEnd);
    SYM(GetErrorString);
#undef SYM
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllReduce && n.AllGather && n.Send && n.Recv &&
           n.GroupStart && n.GroupEnd && n.GetErrorString;
  });
  return n;
}

}  // namespace

struct lod_comm {
  ncclComm_t c = nullptr;
  int nranks = 0, rank = 0, device = 0;
};

#define NCCL_CK(expr)                                                                    \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess) return fail(LOD_ECUDA, "NCCL: %s (%s)", nccl().GetErrorString(_r), #expr); \
  } while (0)

static int need_nccl() {
  if (!nccl().ok) return fail(LOD_ECUDA, "NCCL is not available (libnccl.so.2 not found)");
  return LOD_OK;
}

extern "C" {

int lod_comm_unique_id(uint8_t* out128) {
  if (int r = need_nccl()) return r;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  NCCL_CK(nccl().GetUniqueId(&id));
  std::memcpy(out128, &id, 128);
  return LOD_OK;
}

int lod_comm_init(const uint8_t* id128, int nranks, int rank, int device, lod_comm** out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(LOD_EVALUE, "bad communicator arguments");
  if (int r = need_nccl()) return r;
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return fail(LOD_ECUDA, "cannot use CUDA device %d", device);
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  lod_comm* c = new lod_comm();
  ncclResult_t r = nccl().CommInitRank(&c->c, nranks, id, rank);
  if (prev >= 0) cudaSetDevice(prev);
  if (r != ncclSuccess) {
    delete c;
    return fail(LOD_ECUDA, "NCCL: %s (ncclCommInitRank)", nccl().GetErrorString(r));
  }
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  *out = c;
  return LOD_OK;
}

int lod_comm_destroy(lod_comm* c) {
  if (!c) return LOD_OK;
  if (c->c) nccl().CommDestroy(c->c);
  delete c;
  return LOD_OK;
}

int lod_comm_allreduce(lod_comm* c, void* d_buf, uint64_t count, int dtype, int op, void* stream) {
  if (!c) return fail(LOD_EVALUE, "null communicator");
  static const ncclDataType_t types[] = {ncclUint32, ncclUint64, ncclFloat64, ncclInt64};
  static const ncclRedOp_t ops[] = {ncclSum, ncclMin, ncclMax};
  if (dtype < 0 || dtype > 3 || op < 0 || op > 2) return fail(LOD_EVALUE, "bad all-reduce type / op");
  if (!count) return LOD_OK;
  NCCL_CK(nccl().AllReduce(d_buf, d_buf, count, types[dtype], ops[op], c->c, (cudaStream_t)stream));
  return LOD_OK;
}

int lod_comm_allgather(lod_comm* c, const void* d_send, void* d_recv, uint64_t bytes, void* stream) {
  if (!c) return fail(LOD_EVALUE, "null communicator");
  NCCL_CK(nccl().AllGather(d_send, d_recv, bytes, ncclUint8, c->c, (cudaStream_t)stream));
  return LOD_OK;
}

// Point exchange: rank r sends send_bytes[q] bytes (consecutive in d_send, by destination rank)
// to every q and receives recv_bytes[q] from every q into d_recv in SOURCE-rank order -- which
// keeps every leaf's points in global input order (H3).  One NCCL group: all transfers overlap.
int lod_comm_alltoallv(lod_comm* c, const void* d_send, const uint64_t* send_bytes, void* d_recv,
                       const uint64_t* recv_bytes, void* stream) {
  if (!c || !send_bytes || !recv_bytes) return fail(LOD_EVALUE, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t so = 0, ro = 0;
  uint64_t self_so = 0, self_ro = 0;
  NCCL_CK(nccl().GroupStart());
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {  // own part: a device copy
      self_so = so, self_ro = ro;
    } else {
      if (send_bytes[q]) nccl().Send(static_cast<const char*>(d_send) + so, send_bytes[q], ncclUint8, q, c->c, s);
      if (recv_bytes[q]) nccl().Recv(static_cast<char*>(d_recv) + ro, recv_bytes[q], ncclUint8, q, c->c, s);
    }
    so += send_bytes[q];
    ro += recv_bytes[q];
  }
  NCCL_CK(nccl().GroupEnd());
  if (send_bytes[c->rank] != recv_bytes[c->rank]) return fail(LOD_EVALUE, "self send / receive sizes differ");
  if (send_bytes[c->rank] &&
      cudaMemcpyAsync(static_cast<char*>(d_recv) + self_ro, static_cast<const char*>(d_send) + self_so,
                      send_bytes[c->rank], cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(LOD_ECUDA, "all-to-all self copy failed");
  return LOD_OK;
}

// Gather to `root`: every rank sends `bytes`; root receives recv_bytes[q] from each q,
// concatenated in rank order (root's own part copied on the stream).
int lod_comm_gatherv(lod_comm* c, const void* d_send, uint64_t bytes, void* d_recv, const uint64_t* recv_bytes,
                     int root, void* stream) {
  if (!c || root < 0 || root >= c->nranks) return fail(LOD_EVALUE, "bad gather arguments");
  if (c->rank == root && !recv_bytes) return fail(LOD_EVALUE, "root needs recv_bytes");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t self_off = 0;
  NCCL_CK(nccl().GroupStart());
  if (c->rank == root) {
    uint64_t off = 0;
    for (int q = 0; q < c->nranks; ++q) {
      if (q == root) self_off = off;
      else if (recv_bytes[q]) nccl().Recv(static_cast<char*>(d_recv) + off, recv_bytes[q], ncclUint8, q, c->c, s);
      off += recv_bytes[q];
    }
  } else if (bytes) {
    nccl().Send(d_send, bytes, ncclUint8, root, c->c, s);
  }
  NCCL_CK(nccl().GroupEnd());
  if (c->rank == root && bytes &&
      cudaMemcpyAsync(static_cast<char*>(d_recv) + self_off, d_send, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(LOD_ECUDA, "gather self copy failed");
  return LOD_OK;
}

}  // extern "C"
