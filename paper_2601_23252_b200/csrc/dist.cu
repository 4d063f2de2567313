// Multi-GPU transport: one process per GPU.
//
// NS runs shard the live set (k_shard.cu): one in-place NCCL all-gather of a
// fixed-size block per rank per iteration (candidates + moment sums), and the
// ranks' live-set arrays mapped into each other's address space with CUDA IPC
// so the chain kernels read parent rows another rank owns directly over
// NVLink (ipc_exchange).
//
// F3 tempered SMC contexts keep the replicated layout: the HRSS chains are
// split in contiguous blocks of kc = ceil(n / W) per rank and, after its
// chains finish, each rank's new rows (x, E) reach every rank through one
// NCCL all-gather (exchange_chains).
//
// NCCL is loaded with dlopen (the copy PyTorch already mapped, when present),
// so libnss has no link-time dependency on it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nss_internal.cuh"

namespace nss {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
};

const NcclApi *nccl_api() {
  static NcclApi api;
  static int state = 0;  // 0 untried, 1 ok, -1 unavailable
  if (state) return state > 0 ? &api : nullptr;
  const char *env = getenv("NSS_NCCL_LIB");
  const char *names[] = {env, "libnccl.so.2", "libnccl.so"};
  void *h = nullptr;
  for (const char *nm : names)
    if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    state = -1;
    return nullptr;
  }
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  state = (api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy) ? 1 : -1;
  return state > 0 ? &api : nullptr;
}

namespace {

// row of chain c: x (dp floats, zero past d) then E
__global__ void k_pack_chains(RunDev r, float *buf, int row) {
  const int c = r.c0 + blockIdx.x;
  if (c >= r.c1) return;
  const int s = r.cdest[c];
  float *o = buf + static_cast<long long>(c - r.c0) * row;
  for (int i = threadIdx.x; i < row; i += blockDim.x)
    o[i] = i < r.dp ? r.X[static_cast<long long>(s) * r.dp + i] : r.E[s];
}

__global__ void k_unpack_chains(RunDev r, const float *all, int row) {
  const int c = blockIdx.x;
  if (c >= r.nch || (c >= r.c0 && c < r.c1)) return;  // own rows are already in place
  const DevState *st = r.st;
  const int s = r.cdest[c];
  const float *in = all + static_cast<long long>(c) * row;
  for (int i = threadIdx.x; i < row; i += blockDim.x) {
    if (i < r.dp)
      r.X[static_cast<long long>(s) * r.dp + i] = in[i];
    else
      r.E[s] = in[i];
  }
  if (threadIdx.x == 0 && !(st->terminated || st->error || st->finalised) && r.cpar[c] != s) r.birth[s] = st->e_star;
}

}  // namespace

bool nccl_unique_id(uint8_t out[128]) {
  const NcclApi *api = nccl_api();
  if (!api) return false;
  ncclUniqueId id;
  if (api->get_unique_id(&id) != ncclSuccess) return false;
  static_assert(sizeof(id.internal) == 128, "NCCL unique id size");
  memcpy(out, id.internal, 128);
  return true;
}

bool nccl_comm_init(void **comm, int world, const uint8_t uid[128], int rank, std::string *err) {
  const NcclApi *api = nccl_api();
  if (!api) {
    *err = "NCCL library not found (set NSS_NCCL_LIB)";
    return false;
  }
  ncclUniqueId id;
  memcpy(id.internal, uid, 128);
  ncclComm_t c = nullptr;
  const ncclResult_t rc = api->comm_init_rank(&c, world, id, rank);
  if (rc != ncclSuccess) {
    *err = std::string("ncclCommInitRank: ") + (api->error_string ? api->error_string(rc) : "error");
    return false;
  }
  *comm = c;
  return true;
}

void nccl_comm_free(void *comm) {
  const NcclApi *api = nccl_api();
  if (api && comm) api->comm_destroy(static_cast<ncclComm_t>(comm));
}

// In-place all-gather of `bytes` per rank: rank q's block at buf + q * bytes.
bool nccl_allgather_inplace(void *comm, void *buf, size_t bytes, int rank, cudaStream_t stream, std::string *err) {
  const NcclApi *api = nccl_api();
  char *b = static_cast<char *>(buf);
  const ncclResult_t rc = api->all_gather(b + static_cast<size_t>(rank) * bytes, b, bytes, ncclUint8,
                                          static_cast<ncclComm_t>(comm), stream);
  if (rc != ncclSuccess) {
    *err = std::string("ncclAllGather: ") + (api->error_string ? api->error_string(rc) : "error");
    return false;
  }
  return true;
}

// CUDA IPC handles of this rank's arrays (nptr of them, cudaMalloc'd) to every
// rank; peers[i * world + q] = rank q's i-th array mapped here (own: local).
bool ipc_exchange(void *comm, int world, int rank, void *const *mine, int nptr, void **peers,
                  std::vector<void *> *opened, cudaStream_t stream, std::string *err) {
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  const size_t blk = ((hb * nptr) + 255) & ~static_cast<size_t>(255);
  std::vector<char> host(blk * world, 0);
  for (int i = 0; i < nptr; ++i) {
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, mine[i]) != cudaSuccess) {
      *err = "cudaIpcGetMemHandle failed";
      return false;
    }
    memcpy(host.data() + rank * blk + i * hb, &h, hb);
  }
  char *dev = nullptr;
  if (cudaMalloc(&dev, blk * world) != cudaSuccess) {
    *err = "cudaMalloc (ipc exchange)";
    return false;
  }
  bool ok = cudaMemcpyAsync(dev + rank * blk, host.data() + rank * blk, blk, cudaMemcpyHostToDevice, stream) ==
                cudaSuccess &&
            nccl_allgather_inplace(comm, dev, blk, rank, stream, err) &&
            cudaMemcpyAsync(host.data(), dev, blk * world, cudaMemcpyDeviceToHost, stream) == cudaSuccess &&
            cudaStreamSynchronize(stream) == cudaSuccess;
  cudaFree(dev);
  if (!ok) {
    if (err->empty()) *err = "ipc handle exchange failed";
    return false;
  }
  for (int i = 0; i < nptr; ++i)
    for (int q = 0; q < world; ++q) {
      if (q == rank) {
        peers[i * world + q] = mine[i];
        continue;
      }
      cudaIpcMemHandle_t h;
      memcpy(&h, host.data() + q * blk + i * hb, hb);
      void *p = nullptr;
      if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        *err = "cudaIpcOpenMemHandle failed (no peer access between the ranks' GPUs?)";
        return false;
      }
      opened->push_back(p);
      peers[i * world + q] = p;
    }
  return true;
}

// pack this rank's chain rows, all-gather kc rows per rank, scatter all k rows
bool exchange_chains(const RunDev &r, void *comm, float *buf, float *all, int kc, const LaunchCtx &lc,
                     std::string *err) {
  const int row = r.dp + 1;
  k_pack_chains<<<kc > 0 ? kc : 1, 128, 0, lc.stream>>>(r, buf, row);
  ++*lc.launch_counter;
  const ncclResult_t rc = nccl_api()->all_gather(buf, all, static_cast<size_t>(kc) * row, ncclFloat32,
                                                 static_cast<ncclComm_t>(comm), lc.stream);
  if (rc != ncclSuccess) {
    *err = std::string("ncclAllGather: ") + (nccl_api()->error_string ? nccl_api()->error_string(rc) : "error");
    return false;
  }
  k_unpack_chains<<<r.nch, 128, 0, lc.stream>>>(r, all, row);
  ++*lc.launch_counter;
  return true;
}

}  // namespace nss
