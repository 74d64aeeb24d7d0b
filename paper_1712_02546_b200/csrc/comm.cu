// comm.cu — the two collectives the kernel split creates, over NCCL on NVLink/NVSwitch.
//
//  * forward: channel AllGather of the per-rank output blocks (the paper's gather +
//    "reshapes and rearranges", Alg. 1 L19-22).  Because the gather
//    layout stores each rank's channels as one contiguous block in rank order, equal
//    block widths make this ONE in-place ncclAllGather; unequal widths (Eq. 1 maps) are a
//    grouped set of ncclBroadcast calls, one per root (allgather-v).
//  * backward: sum of the per-rank partial dX (north_star) as in-place ncclAllReduce, or
//    ncclReduceScatter delivering each rank exactly its own input block (grouped
//    ncclReduce per root for unequal widths).
#include <nccl.h>

#include <string>
#include <vector>

#include "kernels.cuh"

#include <cuda.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <functional>
#include <map>

// A symmetric buffer: the same-sized allocation on every rank, each rank holding peer pointers
// (CUDA IPC over NVLink) to all the others, so kernels can store directly into peers' copies.
struct SymBuf {
  size_t bytes, flag_off;
  int64_t own_off = -1, own_elems = 0;   // this rank's block (floats), recorded by its producer
  void* peers[CP_MAX_RANKS];  // peers[rank] = own pointer
  int index = -1;             // loopback: allocation sequence number (peers resolved by it)
  // NVLink multicast (CP_MULTICAST=1): the buffer is a driver VMM allocation bound to a multicast
  // object; `mc` maps it (a store / reduction through `mc` reaches every rank's copy via NVSwitch)
  cudaEvent_t pending = nullptr;   // producer's deferred barrier, waited for by the consumer
  bool vmm = false;
  size_t map_bytes = 0;
  void* mc = nullptr;
  CUmemGenericAllocationHandle h[CP_MAX_RANKS] = {}, h_mc = 0;
};

// Loopback group (tests on one GPU): `world` simulated ranks in one process, each with its own
// cp_comm handle.  Symmetric buffers are plain allocations on the current device; the k-th
// allocation of every handle forms one symmetric buffer (peers resolved by index).  No NCCL.
struct LoopGroup {
  int world = 0, alive = 0;
  std::vector<std::vector<void*>> bufs;   // [allocation index][rank]
  std::vector<void*> ctl;                  // control line per rank
  // comm-stream tails of the fused reduce-scatter, enqueued once every rank issued its compute
  std::vector<cudaEvent_t> done;
  std::vector<std::function<int(const std::vector<cudaEvent_t>&)>> pending;
};

struct cp_comm_s {
  ncclComm_t comm;
  int rank, world;
  std::map<void*, SymBuf> sym;   // keyed by the local pointer
  float* barrier_word = nullptr; // 1-float device scratch for the teardown barrier
  // control line (symmetric, u32 words): [0,16) barrier slots written by the peers (their epoch),
  // [16] this rank's barrier epoch, [17] the constant 1 (source of copy-engine flag writes)
  uint32_t* ctl = nullptr;
  uint32_t* ctl_peer[CP_MAX_RANKS] = {};
  // one-shot AllReduce scratch (symmetric): [parity][source rank][kArMax] floats
  float* ar = nullptr;
  float* ar_peer[CP_MAX_RANKS] = {};
  LoopGroup* loop = nullptr;      // loopback handle (cp_comm_create_loopback), else NCCL
  int sym_count = 0;              // loopback: symmetric allocations made through this handle
};
constexpr int kCtlEpoch = 16, kCtlOne = 17, kCtlChunks = 18, kCtlArFlags = 32, kCtlArEpoch = 48, kCtlWords = 64;
constexpr int64_t kArMax = 1 << 16;   // one-shot AllReduce capacity (floats)

#define CP_NCCL(call)                                                                      \
  do {                                                                                     \
    ncclResult_t r__ = (call);                                                             \
    if (r__ != ncclSuccess) {                                                              \
      ::cp::set_error(std::string(#call) + ": " + ncclGetErrorString(r__));               \
      return CP_ERR_NCCL;                                                                  \
    }                                                                                      \
  } while (0)

extern "C" int cp_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) CP_FAIL(CP_ERR_ARG, "cp_comm_unique_id: null pointer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId id;
  CP_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, 128);
  return CP_OK;
}

extern "C" int cp_comm_create(const uint8_t id[128], int32_t rank, int32_t world, cp_comm* out) {
  if (!id || !out) CP_FAIL(CP_ERR_ARG, "cp_comm_create: null pointer");
  if (world < 1 || world > CP_MAX_RANKS || rank < 0 || rank >= world)
    CP_FAIL(CP_ERR_CONFIG, "cp_comm_create: bad rank/world " + std::to_string(rank) + "/" + std::to_string(world));
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  auto* c = new cp_comm_s{};
  c->rank = rank;
  c->world = world;
  ncclResult_t r = ncclCommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    CP_FAIL(CP_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *out = c;
  return CP_OK;
}

// P simulated ranks of one process on the current GPU (tests of the fused peer-memory paths).
extern "C" int cp_comm_create_loopback(int32_t world, cp_comm* out) {
  if (!out) CP_FAIL(CP_ERR_ARG, "cp_comm_create_loopback: null pointer");
  if (world < 1 || world > CP_MAX_RANKS) CP_FAIL(CP_ERR_CONFIG, "cp_comm_create_loopback: world out of [1,16]");
  auto* g = new LoopGroup{};
  g->world = world;
  g->alive = world;
  g->ctl.assign(world, nullptr);
  for (int r = 0; r < world; ++r) {
    auto* c = new cp_comm_s{};
    c->comm = nullptr;
    c->rank = r;
    c->world = world;
    c->loop = g;
    out[r] = c;
  }
  return CP_OK;
}

static int sym_map(cp_comm c, size_t bytes, void** local_out, SymBuf& sb);
static int sym_map_multicast(cp_comm c, size_t bytes, void** local_out, SymBuf& sb, bool* done);
namespace cp { bool multicast_requested(); }
using cp::multicast_requested;

extern "C" int cp_symmetric_alloc(cp_comm c, size_t bytes, void** local_out) {
  if (!c || !local_out || bytes == 0) CP_FAIL(CP_ERR_ARG, "cp_symmetric_alloc: bad arguments");
  if (c->loop) {
    LoopGroup& g = *c->loop;
    if (!c->ctl) {
      void* p = nullptr;
      CP_CUDA(cudaMalloc(&p, kCtlWords * 4));
      CP_CUDA(cudaMemset(p, 0, kCtlWords * 4));
      const uint32_t consts[2] = {1u, (uint32_t)cp::kGatherChunks};
      CP_CUDA(cudaMemcpy((uint32_t*)p + kCtlOne, consts, 8, cudaMemcpyHostToDevice));
      c->ctl = (uint32_t*)p;
      g.ctl[c->rank] = p;
    }
    SymBuf sb{};
    sb.bytes = bytes;
    sb.flag_off = (bytes + 255) / 256 * 256;
    void* mine = nullptr;
    CP_CUDA(cudaMalloc(&mine, sb.flag_off + 256));
    CP_CUDA(cudaMemset(mine, 0, sb.flag_off + 256));
    sb.index = c->sym_count++;
    if ((int)g.bufs.size() <= sb.index) g.bufs.resize(sb.index + 1, std::vector<void*>(g.world, nullptr));
    g.bufs[sb.index][c->rank] = mine;
    for (int q = 0; q < c->world; ++q) sb.peers[q] = q == c->rank ? mine : nullptr;   // resolved on use
    c->sym[mine] = sb;
    *local_out = mine;
    return CP_OK;
  }
  if (!c->ctl) {   // first symmetric allocation (collective): the control line
    SymBuf cb{};
    void* p = nullptr;
    CP_TRY(sym_map(c, kCtlWords * 4, &p, cb));
    c->ctl = (uint32_t*)p;
    for (int q = 0; q < c->world; ++q) c->ctl_peer[q] = (uint32_t*)cb.peers[q];
    const uint32_t consts[2] = {1u, (uint32_t)cp::kGatherChunks};
    CP_CUDA(cudaMemcpy(c->ctl + kCtlOne, consts, 8, cudaMemcpyHostToDevice));
  }
  SymBuf sb{};
  bool done = false;
  if (multicast_requested()) CP_TRY(sym_map_multicast(c, bytes, local_out, sb, &done));
  if (!done) CP_TRY(sym_map(c, bytes, local_out, sb));
  c->sym[*local_out] = sb;
  return CP_OK;
}

// All-gather `n` bytes per rank through NCCL (blocking; allocation time only).  Also a barrier.
static int allgather_bytes(cp_comm c, const void* mine, size_t n, std::vector<uint8_t>& all) {
  uint8_t* dev = nullptr;
  CP_CUDA(cudaMalloc(&dev, n * (size_t)(c->world + 1)));
  CP_CUDA(cudaMemcpy(dev + n * (size_t)c->world, mine, n, cudaMemcpyHostToDevice));
  ncclResult_t r = ncclAllGather(dev + n * (size_t)c->world, dev, n, ncclUint8, c->comm, 0);
  all.assign(n * (size_t)c->world, 0);
  cudaError_t e = cudaSuccess;
  if (r == ncclSuccess) e = cudaMemcpy(all.data(), dev, all.size(), cudaMemcpyDeviceToHost);
  cudaFree(dev);
  if (r != ncclSuccess) CP_FAIL(CP_ERR_NCCL, std::string("symmetric alloc exchange: ") + ncclGetErrorString(r));
  if (e != cudaSuccess) CP_FAIL(CP_ERR_CUDA, std::string("symmetric alloc exchange: ") + cudaGetErrorString(e));
  return CP_OK;
}

// allocate + zero `bytes` (+ a 256 B flag line), exchange IPC handles, map every peer's copy
static int sym_map(cp_comm c, size_t bytes, void** local_out, SymBuf& sb) {
  sb.bytes = bytes;
  sb.flag_off = (bytes + 255) / 256 * 256;   // arrival flags live behind the data (one 256 B line)
  void* mine = nullptr;
  CP_CUDA(cudaMalloc(&mine, sb.flag_off + 256));
  CP_CUDA(cudaMemset(mine, 0, sb.flag_off + 256));
  cudaIpcMemHandle_t h;
  CP_CUDA(cudaIpcGetMemHandle(&h, mine));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::vector<uint8_t> all;
  CP_TRY(allgather_bytes(c, &h, 64, all));
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank) {
      sb.peers[p] = mine;
      continue;
    }
    cudaIpcMemHandle_t ph;
    memcpy(&ph, all.data() + 64 * (size_t)p, 64);
    CP_CUDA(cudaIpcOpenMemHandle(&sb.peers[p], ph, cudaIpcMemLazyEnablePeerAccess));
  }
  if (!c->barrier_word) {
    CP_CUDA(cudaMalloc(&c->barrier_word, sizeof(float)));
    CP_CUDA(cudaMemset(c->barrier_word, 0, sizeof(float)));
  }
  *local_out = mine;
  return CP_OK;
}

// ---------------------------------------------------------------------------------------------
// NVLink multicast symmetric buffers (CP_MULTICAST=1).  Driver VMM: each rank cuMemCreate's its
// copy with a POSIX-fd shareable handle; peers obtain the exporter's fd with pidfd_getfd (same node,
// same user) and map it; rank 0 creates the multicast object, every rank adds its device and binds
// its copy, and maps the multicast address.  Driver entry points come from cudaGetDriverEntryPoint
// (no libcuda link).  Any failure on any rank is agreed collectively and the buffer falls back to
// the CUDA-IPC path above, so every rank always takes the same path.
struct Drv {
  bool ok = false;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*memRelease)(CUmemGenericAllocationHandle);
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*addrFree)(CUdeviceptr, size_t);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*exportH)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
  CUresult (*importH)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long);
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
};
static Drv& drv() {
  static Drv d = [] {
    Drv x{};
    bool ok = true;
    auto get = [&](const char* name, auto& fn) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
          !p)
        ok = false;
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
    };
    get("cuMemCreate", x.memCreate);
    get("cuMemRelease", x.memRelease);
    get("cuMemGetAllocationGranularity", x.granularity);
    get("cuMemAddressReserve", x.reserve);
    get("cuMemAddressFree", x.addrFree);
    get("cuMemMap", x.map);
    get("cuMemUnmap", x.unmap);
    get("cuMemSetAccess", x.setAccess);
    get("cuMemExportToShareableHandle", x.exportH);
    get("cuMemImportFromShareableHandle", x.importH);
    get("cuMulticastCreate", x.mcCreate);
    get("cuMulticastAddDevice", x.mcAddDevice);
    get("cuMulticastBindMem", x.mcBindMem);
    get("cuMulticastUnbind", x.mcUnbind);
    get("cuMulticastGetGranularity", x.mcGranularity);
    x.ok = ok;
    return x;
  }();
  return d;
}

bool cp::multicast_requested() {
  static const int v = [] {
    const char* e = getenv("CP_MULTICAST");
    return e ? atoi(e) : 0;
  }();
  return v != 0;
}

// reserve + map + grant this device read/write access
static bool vmm_map(CUmemGenericAllocationHandle h, size_t size, size_t align, int dev, void** va_out) {
  Drv& d = drv();
  CUdeviceptr va = 0;
  if (d.reserve(&va, size, align, 0, 0) != CUDA_SUCCESS) return false;
  if (d.map(va, size, 0, h, 0) != CUDA_SUCCESS) {
    d.addrFree(va, size);
    return false;
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (d.setAccess(va, size, &acc, 1) != CUDA_SUCCESS) {
    d.unmap(va, size);
    d.addrFree(va, size);
    return false;
  }
  *va_out = (void*)va;
  return true;
}

static void vmm_unmap(void* va, size_t size) {
  if (!va) return;
  drv().unmap((CUdeviceptr)va, size);
  drv().addrFree((CUdeviceptr)va, size);
}

// a peer process's file descriptor, duplicated into this process (Linux >= 5.6)
static int fd_from_peer(int pid, int fd) {
#if defined(SYS_pidfd_open) && defined(SYS_pidfd_getfd)
  const int pfd = (int)syscall(SYS_pidfd_open, pid, 0);
  if (pfd < 0) return -1;
  const int mine = (int)syscall(SYS_pidfd_getfd, pfd, fd, 0);
  close(pfd);
  return mine;
#else
  (void)pid;
  (void)fd;
  return -1;
#endif
}

// collective: every rank contributes `ok`; true iff all ranks are ok
static int agree(cp_comm c, bool ok, bool* all_ok) {
  const uint8_t v = ok ? 1 : 0;
  std::vector<uint8_t> all;
  CP_TRY(allgather_bytes(c, &v, 1, all));
  *all_ok = true;
  for (uint8_t a : all) *all_ok = *all_ok && a;
  return CP_OK;
}

static void vmm_release(cp_comm c, SymBuf& sb) {
  Drv& d = drv();
  int dev = 0;
  cudaGetDevice(&dev);
  if (sb.mc) vmm_unmap(sb.mc, sb.map_bytes);
  if (sb.h_mc) {
    if (sb.h[c->rank]) d.mcUnbind(sb.h_mc, dev, 0, sb.map_bytes);
    d.memRelease(sb.h_mc);
  }
  for (int q = 0; q < c->world; ++q) {
    if (sb.peers[q]) vmm_unmap(sb.peers[q], sb.map_bytes);
    if (sb.h[q]) d.memRelease(sb.h[q]);
    sb.peers[q] = nullptr;
    sb.h[q] = 0;
  }
  sb.mc = nullptr;
  sb.h_mc = 0;
}

// Returns CP_OK with *done=false (nothing allocated) if any rank could not set the buffer up.
static int sym_map_multicast(cp_comm c, size_t bytes, void** local_out, SymBuf& sb, bool* done) {
  *done = false;
  Drv& d = drv();
  int dev = 0;
  CP_CUDA(cudaGetDevice(&dev));
  sb.bytes = bytes;
  sb.flag_off = (bytes + 255) / 256 * 256;
  sb.vmm = true;
  const int me = c->rank;
  bool ok = d.ok;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)c->world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g1 = 0, g2 = 0;
  if (ok) ok = d.granularity(&g1, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS;
  if (ok) ok = d.mcGranularity(&g2, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS;
  const size_t gran = std::max<size_t>(std::max(g1, g2), 1);
  const size_t size = (sb.flag_off + 256 + gran - 1) / gran * gran;
  sb.map_bytes = size;
  mp.size = size;
  int fds[3] = {(int)getpid(), -1, -1};   // pid, fd of this rank's copy, fd of the multicast object (rank 0)
  if (ok) ok = d.memCreate(&sb.h[me], size, &prop, 0) == CUDA_SUCCESS;
  if (ok) ok = vmm_map(sb.h[me], size, gran, dev, &sb.peers[me]);
  if (ok) ok = cudaMemset(sb.peers[me], 0, size) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
  if (ok) ok = d.exportH(&fds[1], sb.h[me], CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) == CUDA_SUCCESS;
  if (ok && me == 0) {
    ok = d.mcCreate(&sb.h_mc, &mp) == CUDA_SUCCESS;
    if (ok) ok = d.exportH(&fds[2], sb.h_mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) == CUDA_SUCCESS;
  }
  std::vector<uint8_t> all;
  bool all_ok = false;
  int rc = agree(c, ok, &all_ok);
  if (rc == CP_OK && all_ok) rc = allgather_bytes(c, fds, sizeof(fds), all);
  if (rc == CP_OK && all_ok) {
    // import the peers' copies and (ranks > 0) the multicast object
    auto peer_fds = [&](int q, int k) {
      int v;
      memcpy(&v, all.data() + sizeof(fds) * (size_t)q + 4 * k, 4);
      return v;
    };
    for (int q = 0; q < c->world && ok; ++q) {
      if (q == me) continue;
      const int fd = fd_from_peer(peer_fds(q, 0), peer_fds(q, 1));
      ok = fd >= 0 && d.importH(&sb.h[q], (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) == CUDA_SUCCESS;
      if (fd >= 0) close(fd);
      if (ok) ok = vmm_map(sb.h[q], size, gran, dev, &sb.peers[q]);
    }
    if (ok && me != 0) {
      const int fd = fd_from_peer(peer_fds(0, 0), peer_fds(0, 2));
      ok = fd >= 0 && d.importH(&sb.h_mc, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) == CUDA_SUCCESS;
      if (fd >= 0) close(fd);
    }
    if (ok) ok = d.mcAddDevice(sb.h_mc, dev) == CUDA_SUCCESS;
    rc = agree(c, ok, &all_ok);   // every device added before any bind; exporters may close their fds
  }
  if (fds[1] >= 0) close(fds[1]);
  if (fds[2] >= 0) close(fds[2]);
  if (rc == CP_OK && all_ok) {
    ok = d.mcBindMem(sb.h_mc, 0, sb.h[me], 0, size, 0) == CUDA_SUCCESS;
    rc = agree(c, ok, &all_ok);
  }
  if (rc == CP_OK && all_ok) {
    ok = vmm_map(sb.h_mc, size, gran, dev, &sb.mc);
    rc = agree(c, ok, &all_ok);
  }
  if (rc != CP_OK || !all_ok) {
    vmm_release(c, sb);
    sb = SymBuf{};
    if (rc != CP_OK) return rc;
    return CP_OK;   // *done = false: the caller falls back to CUDA IPC
  }
  if (!c->barrier_word) {
    CP_CUDA(cudaMalloc(&c->barrier_word, sizeof(float)));
    CP_CUDA(cudaMemset(c->barrier_word, 0, sizeof(float)));
  }
  *local_out = sb.peers[me];
  *done = true;
  return CP_OK;
}

// Unmap every peer's copy, then wait until all ranks have unmapped theirs before freeing the
// exported allocation (no rank may still hold a mapping of memory that is being freed).
static void sym_release(cp_comm c, void* local, SymBuf& sb) {
  cudaDeviceSynchronize();
  if (c->loop) {   // simulated ranks: no mappings, no cross-rank barrier
    if (sb.index >= 0 && sb.index < (int)c->loop->bufs.size()) c->loop->bufs[sb.index][c->rank] = nullptr;
    cudaFree(local);
    return;
  }
  if (sb.vmm) {   // multicast: unbind + unmap everything, then the barrier, then the own copy
    Drv& d = drv();
    int dev = 0;
    cudaGetDevice(&dev);
    if (sb.mc) vmm_unmap(sb.mc, sb.map_bytes);
    if (sb.h_mc) d.mcUnbind(sb.h_mc, dev, 0, sb.map_bytes);
    for (int p = 0; p < c->world; ++p)
      if (p != c->rank) {
        vmm_unmap(sb.peers[p], sb.map_bytes);
        if (sb.h[p]) d.memRelease(sb.h[p]);
      }
  } else {
    for (int p = 0; p < c->world; ++p)
      if (p != c->rank && sb.peers[p]) cudaIpcCloseMemHandle(sb.peers[p]);
  }
  if (c->barrier_word && ncclAllReduce(c->barrier_word, c->barrier_word, 1, ncclFloat, ncclSum, c->comm, 0) ==
                             ncclSuccess)
    cudaDeviceSynchronize();
  if (sb.vmm) {
    if (sb.h_mc) drv().memRelease(sb.h_mc);
    vmm_unmap(local, sb.map_bytes);
    drv().memRelease(sb.h[c->rank]);
    return;
  }
  cudaFree(local);
}

extern "C" int cp_symmetric_free(cp_comm c, void* local) {
  if (!c || !local) return CP_OK;
  auto it = c->sym.find(local);
  if (it == c->sym.end()) CP_FAIL(CP_ERR_ARG, "cp_symmetric_free: not a symmetric buffer");
  sym_release(c, local, it->second);
  c->sym.erase(it);
  return CP_OK;
}

extern "C" int cp_comm_destroy(cp_comm c) {
  if (!c) return CP_OK;
  if (c->loop) {
    for (auto& kv : c->sym) sym_release(c, kv.first, kv.second);
    c->sym.clear();
    if (c->ctl) cudaFree(c->ctl);
    c->loop->ctl[c->rank] = nullptr;
    if (--c->loop->alive == 0) delete c->loop;
    delete c;
    return CP_OK;
  }
  // every rank holds the same number of symmetric buffers, so the per-buffer barriers pair up
  for (auto& kv : c->sym) sym_release(c, kv.first, kv.second);
  c->sym.clear();
  if (c->ar) {
    SymBuf ab{};
    for (int q = 0; q < c->world; ++q) ab.peers[q] = c->ar_peer[q];
    sym_release(c, c->ar, ab);
  }
  if (c->ctl) {
    SymBuf cb{};
    for (int q = 0; q < c->world; ++q) cb.peers[q] = c->ctl_peer[q];
    sym_release(c, c->ctl, cb);
  }
  if (c->barrier_word) cudaFree(c->barrier_word);
  ncclResult_t r = ncclCommDestroy(c->comm);
  delete c;
  if (r != ncclSuccess) CP_FAIL(CP_ERR_NCCL, std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  return CP_OK;
}

// Rank `rank`'s copy of a symmetric buffer and its arrival-flag line, as addressable from this
// process (the local copy, a CUDA-IPC mapping of a peer's, or a simulated rank's allocation).
extern "C" int cp_symmetric_peer(cp_comm c, void* local, int32_t rank, void** data, uint32_t** flags) {
  if (!c || !local || !data || rank < 0 || rank >= c->world) CP_FAIL(CP_ERR_ARG, "cp_symmetric_peer: bad arguments");
  void* peers[CP_MAX_RANKS];
  uint32_t* fl[CP_MAX_RANKS];
  if (c->world == 1) {
    auto it = c->sym.find(local);
    if (it == c->sym.end()) CP_FAIL(CP_ERR_ARG, "cp_symmetric_peer: not a symmetric buffer");
    *data = local;
    if (flags) *flags = (uint32_t*)((char*)local + it->second.flag_off);
    return CP_OK;
  }
  if (!cp::comm_symmetric_peers(c, local, peers, fl))
    CP_FAIL(CP_ERR_ARG, "cp_symmetric_peer: not a symmetric buffer (or a simulated rank has not allocated it yet)");
  *data = peers[rank];
  if (flags) *flags = fl[rank];
  return CP_OK;
}

extern "C" int cp_symmetric_wait(cp_comm c, void* local, void* stream) {
  if (!c || c->world == 1) return CP_OK;
  if (c->loop) CP_FAIL(CP_ERR_UNSUPPORTED, "cp_symmetric_wait: not available on a loopback communicator");
  void* peers[CP_MAX_RANKS];
  uint32_t* flags[CP_MAX_RANKS];
  if (!cp::comm_symmetric_peers(c, local, peers, flags)) CP_FAIL(CP_ERR_ARG, "cp_symmetric_wait: not a symmetric buffer");
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaEvent_t pe = cp::comm_symmetric_take_pending(c, local)) CP_CUDA(cudaStreamWaitEvent(s, pe, 0));
  if (!cp::gather_push_in_epilogue()) CP_TRY(cp::comm_ce_distribute(c, local, s));
  CP_TRY(cp::launch_wait_flags(flags[c->rank], c->world, c->rank, s));
  CP_CUDA(cudaMemsetAsync(flags[c->rank], 0, CP_MAX_RANKS * sizeof(uint32_t), s));
  return CP_OK;
}

// One-shot AllReduce of a small vector over NVLink peer memory (one CTA): write the vector into
// slot [rank] of every rank's scratch (parity = epoch & 1, so the next call cannot overwrite slots
// still being summed: a rank two calls ahead would need this rank's flag of the call in between),
// raise the epoch flag at every peer, wait for all peers' flags, then sum the slots in ascending
// rank order - bitwise identical on every rank.
struct ArPtrs {
  float* s[CP_MAX_RANKS];
  uint32_t* c[CP_MAX_RANKS];
};
// Optional softmax-xent epilogue (y != nullptr): the summed vector is the [B][O] logits; the same block
// then computes loss and dlogits (cp_allreduce_softmax_xent - one launch instead of two).
struct SoftmaxArgs {
  const int* y;
  int B, O;
  float* loss;
  float* dl;
};
__global__ void __launch_bounds__(512) oneshot_allreduce_kernel(float* buf, int n, ArPtrs peers, float* mine,
                                                                uint32_t* ctl, int me, int world, SoftmaxArgs sm) {
  __shared__ uint32_t e_s;
  __shared__ float wsum[16];
  if (threadIdx.x == 0) e_s = ctl[kCtlArEpoch] + 1;
  __syncthreads();
  const uint32_t e = e_s;
  const int par = e & 1;
  for (int q = 0; q < world; ++q) {
    float* dst = peers.s[q] + ((int64_t)par * world + me) * kArMax;
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = buf[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) ctl[kCtlArEpoch] = e;
  // one release per peer, in parallel (thread q): the barrier orders every thread's slot stores
  // before thread q's release (fence cumulativity), so no per-thread fence is needed
  if (threadIdx.x < world && (int)threadIdx.x != me) cp::st_release_sys(peers.c[threadIdx.x] + kCtlArFlags + me, e);
  if (threadIdx.x < world && (int)threadIdx.x != me) {
    const long long t0 = clock64();
    while ((int)(cp::ld_acquire_sys(ctl + kCtlArFlags + threadIdx.x) - e) < 0) {
      asm volatile("nanosleep.u32 32;");
      if (clock64() - t0 > (1ll << 35)) __trap();
    }
  }
  __syncthreads();
  const float* src = mine + (int64_t)par * world * kArMax;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    float t = src[i];
    for (int q = 1; q < world; ++q) t += src[(int64_t)q * kArMax + i];
    buf[i] = t;
  }
  if (sm.y) {
    __syncthreads();   // every summed logit written (block-visible global stores)
    cp::softmax_xent_block(buf, sm.y, sm.B, sm.O, sm.loss, sm.dl, wsum);
  }
}

// Low-latency variant (default for n <= kArMax / 2): every value travels with its epoch in ONE 64-bit word
// (value bits | epoch << 32, single-copy atomic), so a reader polls the data itself - no system fence, no
// separate flag release / acquire round trip.  Slots are double-buffered by epoch parity as above; the
// sum over source ranks runs in ascending rank order: bitwise the same result as the flagged kernel.
constexpr int64_t kArLL = kArMax / 2;   // 64-bit slots per (parity, source rank)
__global__ void __launch_bounds__(512) oneshot_allreduce_ll_kernel(float* buf, int n, ArPtrs peers, float* mine,
                                                                   uint32_t* ctl, int me, int world, SoftmaxArgs sm) {
  __shared__ uint32_t e_s;
  __shared__ float wsum[16];
  if (threadIdx.x == 0) e_s = ctl[kCtlArEpoch] + 1;
  __syncthreads();
  const uint32_t e = e_s;
  const int par = e & 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long w = (unsigned long long)__float_as_uint(buf[i]) | ((unsigned long long)e << 32);
    for (int q = 0; q < world; ++q) {
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(peers.s[q]) + ((int64_t)par * world + me) * kArLL + i;
      asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(dst), "l"(w) : "memory");
    }
  }
  if (threadIdx.x == 0) ctl[kCtlArEpoch] = e;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(mine) + (int64_t)par * world * kArLL;
  const long long t0 = clock64();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    float t = 0.f;
    for (int q = 0; q < world; ++q) {
      unsigned long long w;
      for (;;) {
        asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(w) : "l"(src + (int64_t)q * kArLL + i) : "memory");
        if ((uint32_t)(w >> 32) == e) break;
        if (clock64() - t0 > (1ll << 35)) __trap();
      }
      const float v = __uint_as_float((uint32_t)w);
      t = q == 0 ? v : t + v;
    }
    buf[i] = t;
  }
  if (sm.y) {
    __syncthreads();   // every summed logit written (block-visible global stores)
    cp::softmax_xent_block(buf, sm.y, sm.B, sm.O, sm.loss, sm.dl, wsum);
  }
}

static bool ar_low_latency(int64_t n) {
  static const int on = [] {
    const char* e = getenv("CP_AR_LL");
    return e ? atoi(e) : 1;
  }();
  return on && n <= kArLL;
}

// the one-shot path (scratch allocated lazily, outside graph capture), or nullptr
static float* oneshot_scratch(cp_comm c, int64_t n, cudaStream_t s) {
  if (!c->ctl || n > kArMax) return nullptr;
  if (!c->ar) {   // collective lazy allocation - not while a graph is being captured
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) return nullptr;
    SymBuf ab{};
    void* p = nullptr;
    if (sym_map(c, (size_t)2 * c->world * kArMax * 4, &p, ab) != CP_OK) return nullptr;
    c->ar = (float*)p;
    for (int q = 0; q < c->world; ++q) c->ar_peer[q] = (float*)ab.peers[q];
  }
  return c->ar;
}

extern "C" int cp_allreduce_sum(cp_comm c, float* buf, int64_t n, void* stream) {
  if (!c || c->world == 1 || n == 0) return CP_OK;
  if (!buf || n < 0) CP_FAIL(CP_ERR_ARG, "cp_allreduce_sum: bad arguments");
  if (c->loop) CP_FAIL(CP_ERR_UNSUPPORTED, "cp_allreduce_sum: not available on a loopback communicator");
  cudaStream_t s = (cudaStream_t)stream;
  if (oneshot_scratch(c, n, s)) {
    ArPtrs ap{};
    for (int q = 0; q < c->world; ++q) {
      ap.s[q] = c->ar_peer[q];
      ap.c[q] = c->ctl_peer[q];
    }
    if (ar_low_latency(n))
      oneshot_allreduce_ll_kernel<<<1, 512, 0, s>>>(buf, (int)n, ap, c->ar, c->ctl, c->rank, c->world, SoftmaxArgs{});
    else
      oneshot_allreduce_kernel<<<1, 512, 0, s>>>(buf, (int)n, ap, c->ar, c->ctl, c->rank, c->world, SoftmaxArgs{});
    CP_LAUNCHED();
    return CP_OK;
  }
  CP_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclFloat, ncclSum, c->comm, s));
  return CP_OK;
}

extern "C" int cp_allreduce_softmax_xent(cp_comm c, float* logits, const int32_t* labels, int32_t B, int32_t O,
                                         float* loss, float* dlogits, void* stream) {
  if (!logits || !labels || !loss || !dlogits || B < 1 || B > 8192 || O < 1 || O > cp::kHeadMaxO)
    CP_FAIL(CP_ERR_ARG, "cp_allreduce_softmax_xent: bad arguments");
  const int64_t n = (int64_t)B * O;
  cudaStream_t s = (cudaStream_t)stream;
  if (c && c->world > 1 && !c->loop && oneshot_scratch(c, n, s)) {
    ArPtrs ap{};
    for (int q = 0; q < c->world; ++q) {
      ap.s[q] = c->ar_peer[q];
      ap.c[q] = c->ctl_peer[q];
    }
    const SoftmaxArgs sm{labels, B, O, loss, dlogits};
    if (ar_low_latency(n))
      oneshot_allreduce_ll_kernel<<<1, 512, 0, s>>>(logits, (int)n, ap, c->ar, c->ctl, c->rank, c->world, sm);
    else
      oneshot_allreduce_kernel<<<1, 512, 0, s>>>(logits, (int)n, ap, c->ar, c->ctl, c->rank, c->world, sm);
    CP_LAUNCHED();
    return CP_OK;
  }
  CP_TRY(cp_allreduce_sum(c, logits, n, stream));   // world 1: no-op; otherwise NCCL (or unsupported)
  return cp_softmax_xent(logits, labels, B, O, loss, dlogits, stream);
}

namespace cp {

static int async_error(cp_comm c) {
  ncclResult_t ar;
  CP_NCCL(ncclCommGetAsyncError(c->comm, &ar));
  if (ar != ncclSuccess) CP_FAIL(CP_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
  return CP_OK;
}

// Every rank must hold the same partition maps: compare min and max of a hash.
int comm_check_plan(cp_comm c, const Layer& L) {
  if (!c || c->world == 1) return CP_OK;
  if (c->world != L.d.world || c->rank != L.d.rank)
    CP_FAIL(CP_ERR_CONFIG, "conv_part_create: desc rank/world " + std::to_string(L.d.rank) + "/" +
                               std::to_string(L.d.world) + " vs communicator " + std::to_string(c->rank) +
                               "/" + std::to_string(c->world));
  if (c->loop) return CP_OK;   // simulated ranks: the caller builds every rank's map itself
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](int64_t v) { h = (h ^ (uint64_t)v) * 1099511628211ull; };
  const cp_partition* ps[2] = {&L.d.out_part, &L.d.in_part};
  for (int t = 0; t < (L.images ? 1 : 2); ++t) {
    mix(ps[t]->n_ranks);
    mix(ps[t]->num_k);
    for (int r = 0; r < ps[t]->n_ranks; ++r) {
      mix(ps[t]->k_begin[r]);
      mix(ps[t]->k_count[r]);
      mix(ps[t]->k_width[r]);
    }
  }
  mix(L.B); mix(L.C); mix(L.H); mix(L.W); mix(L.K); mix(L.R); mix(L.S); mix(L.d.math);
  // split into two non-negative int64 halves so min/max comparisons are exact
  int64_t host[4] = {(int64_t)(h >> 32), (int64_t)(h & 0xffffffffu), -(int64_t)(h >> 32), -(int64_t)(h & 0xffffffffu)};
  int64_t* dev = nullptr;
  CP_CUDA(cudaMalloc(&dev, sizeof(host)));
  CP_CUDA(cudaMemcpy(dev, host, sizeof(host), cudaMemcpyHostToDevice));
  // max over ranks of (h, -h) == (h, -h) on every rank  <=>  all equal
  ncclResult_t r = ncclAllReduce(dev, dev, 4, ncclInt64, ncclMax, c->comm, 0);
  int64_t got[4];
  cudaError_t e = cudaSuccess;
  if (r == ncclSuccess) e = cudaMemcpy(got, dev, sizeof(got), cudaMemcpyDeviceToHost);
  cudaFree(dev);
  if (r != ncclSuccess) CP_FAIL(CP_ERR_NCCL, std::string("plan check: ") + ncclGetErrorString(r));
  if (e != cudaSuccess) CP_FAIL(CP_ERR_CUDA, std::string("plan check: ") + cudaGetErrorString(e));
  for (int i = 0; i < 4; ++i)
    if (got[i] != host[i]) CP_FAIL(CP_ERR_CONFIG, "conv_part_create: ranks hold different partition maps");
  return CP_OK;
}

// Peer pointers of a symmetric buffer (nullptr if `local` is not one).
void comm_symmetric_set_own(cp_comm c, const void* local, int64_t off, int64_t elems) {
  auto it = c->sym.find(const_cast<void*>(local));
  if (it == c->sym.end()) return;
  it->second.own_off = off;
  it->second.own_elems = elems;
}

// Copy-engine gather (consumers outside the tensor-core forward): this rank's block into every
// peer's copy, then the arrival flag (value 1) behind the data at every peer - no SM involved.
int comm_ce_distribute(cp_comm c, const void* local, cudaStream_t s, bool chunks, cudaStream_t s2,
                       const cudaEvent_t* evs) {
  auto it = c->sym.find(const_cast<void*>(local));
  if (it == c->sym.end()) CP_FAIL(CP_ERR_ARG, "not a symmetric buffer");
  const SymBuf& sb = it->second;
  if (sb.own_off < 0) CP_FAIL(CP_ERR_STATE, "symmetric gather: no producer wrote this buffer yet");
  // peers in the order they consume this block (peer q walks its input blocks from its own upwards,
  // so it needs this rank's block after (rank - q) mod P blocks): the soonest consumer first.  With a
  // second stream s2, each peer's copy is split in two halves on two copy engines (the flag follows
  // both: s waits for evs[d] recorded on s2 after the second half)
  const int64_t h = s2 ? (sb.own_elems / 2 + 3) / 4 * 4 : sb.own_elems;   // first half, 16-byte multiple
  for (int d = 1; d < c->world; ++d) {
    const int q = (c->rank - d + c->world) % c->world;
    float* dst = (float*)sb.peers[q] + sb.own_off;
    const float* src = (const float*)local + sb.own_off;
    if (h > 0) CP_CUDA(cudaMemcpyAsync(dst, src, (size_t)h * 4, cudaMemcpyDeviceToDevice, s));
    if (s2) {
      if (sb.own_elems > h)
        CP_CUDA(cudaMemcpyAsync(dst + h, src + h, (size_t)(sb.own_elems - h) * 4, cudaMemcpyDeviceToDevice, s2));
      CP_CUDA(cudaEventRecord(evs[d], s2));
      CP_CUDA(cudaStreamWaitEvent(s, evs[d], 0));
    }
    uint32_t* f = (uint32_t*)((char*)sb.peers[q] + sb.flag_off);
    CP_TRY(comm_signal_ce(c, &f, 1, c->rank, s, chunks));
  }
  return CP_OK;
}

bool comm_is_loopback(cp_comm c) { return c && c->loop; }

// Loopback: the comm-stream tail of rank r's fused reduce-scatter waits for the slots every
// simulated rank stores - on one GPU those are later launches of the same process, so the tails
// are held back until every rank issued its compute (`done` recorded after its dgrad + signal),
// then enqueued in rank order behind all of them: no kernel ever waits on a later launch.
int comm_loopback_defer(cp_comm c, cudaEvent_t done, std::function<int(const std::vector<cudaEvent_t>&)> tail) {
  LoopGroup& g = *c->loop;
  g.done.push_back(done);
  g.pending.push_back(std::move(tail));
  if ((int)g.pending.size() < g.world) return CP_OK;
  std::vector<cudaEvent_t> all;
  all.swap(g.done);
  auto fns = std::move(g.pending);
  g.pending.clear();
  for (auto& f : fns) CP_TRY(f(all));
  return CP_OK;
}

void comm_symmetric_set_pending(cp_comm c, const void* local, cudaEvent_t ev) {
  auto it = c->sym.find(const_cast<void*>(local));
  if (it != c->sym.end()) it->second.pending = ev;
}

cudaEvent_t comm_symmetric_take_pending(cp_comm c, const void* local) {
  if (!c) return nullptr;
  auto it = c->sym.find(const_cast<void*>(local));
  if (it == c->sym.end()) return nullptr;
  cudaEvent_t e = it->second.pending;
  it->second.pending = nullptr;
  return e;
}

// Multicast address of a symmetric buffer (nullptr unless it was set up with CP_MULTICAST=1).
void* comm_symmetric_mc(cp_comm c, const void* local) {
  if (!c || c->world == 1 || c->loop) return nullptr;
  auto it = c->sym.find(const_cast<void*>(local));
  return it == c->sym.end() ? nullptr : it->second.mc;
}

bool comm_symmetric_peers(cp_comm c, const void* local, void** peers, uint32_t** flags) {
  if (!c || c->world == 1) return false;
  auto it = c->sym.find(const_cast<void*>(local));
  if (it == c->sym.end()) return false;
  if (c->loop) {   // resolve the other simulated ranks' copies of this allocation
    const int k = it->second.index;
    if (k < 0 || k >= (int)c->loop->bufs.size()) return false;
    for (int q = 0; q < c->world; ++q) {
      if (!c->loop->bufs[k][q]) return false;
      it->second.peers[q] = c->loop->bufs[k][q];
    }
  }
  for (int p = 0; p < c->world; ++p) {
    peers[p] = it->second.peers[p];
    if (flags) flags[p] = (uint32_t*)((char*)it->second.peers[p] + it->second.flag_off);
  }
  return true;
}

// Cross-rank barrier on `s` through the control line: one thread bumps this rank's epoch, writes it
// into every peer's slot [rank] (st.release.sys over NVLink) and spins until every peer's epoch
// reached it.  Every rank calls it equally often, so the epochs pair up; no NCCL kernel, no host.
struct CtlPtrs {
  uint32_t* p[CP_MAX_RANKS];
};
__global__ void flag_barrier_kernel(CtlPtrs peer, uint32_t* mine, int me, int world) {
  // one warp: thread q releases this rank's epoch at peer q and waits for peer q's (in parallel)
  const int q = threadIdx.x;
  const uint32_t e = mine[kCtlEpoch] + 1;
  __syncwarp();
  if (q == 0) mine[kCtlEpoch] = e;
  if (q < world && q != me) {
    st_release_sys(peer.p[q] + me, e);
    const long long t0 = clock64();
    while ((int)(ld_acquire_sys(mine + q) - e) < 0) {
      asm volatile("nanosleep.u32 64;");
      if (clock64() - t0 > (1ll << 35)) __trap();
    }
  }
  __syncwarp();
}

int comm_barrier(cp_comm c, cudaStream_t s) {
  if (!c || c->world == 1) return CP_OK;
  if (c->loop) return CP_OK;   // simulated ranks share one GPU and the caller's stream order
  if (!c->ctl) {
    CP_NCCL(ncclAllReduce(c->barrier_word, c->barrier_word, 1, ncclFloat, ncclSum, c->comm, s));
    return CP_OK;
  }
  CtlPtrs cp{};
  for (int q = 0; q < c->world; ++q) cp.p[q] = c->ctl_peer[q];
  flag_barrier_kernel<<<1, 32, 0, s>>>(cp, c->ctl, c->rank, c->world);
  CP_LAUNCHED();
  return CP_OK;
}

// Arrival flags raised by the copy engines (no SM): 4-byte copies of the constant 1 into slot
// `slot` of each given flag array, ordered after the data copies on the same stream.
int comm_signal_ce(cp_comm c, uint32_t* const* flags, int n, int slot, cudaStream_t s, bool chunks) {
  for (int k = 0; k < n; ++k)
    CP_CUDA(cudaMemcpyAsync(flags[k] + slot, c->ctl + (chunks ? kCtlChunks : kCtlOne), 4,
                            cudaMemcpyDeviceToDevice, s));
  return CP_OK;
}

static bool equal_widths(const Blocks& g) {
  for (int r = 1; r < g.n; ++r)
    if (g.kw[r] != g.kw[0]) return false;
  return true;
}

int comm_allgather_blocks(cp_comm c, float* buf, const Blocks& g, cudaStream_t s) {
  if (!c || c->world == 1) return CP_OK;
  if (c->loop) CP_FAIL(CP_ERR_UNSUPPORTED, "loopback communicator: NCCL collectives unavailable (fused paths only)");
  CP_TRY(async_error(c));
  if (equal_widths(g)) {
    const size_t cnt = (size_t)(g.start[1] - g.start[0]);
    if (cnt == 0) return CP_OK;
    CP_NCCL(ncclAllGather(buf + g.start[c->rank], buf, cnt, ncclFloat, c->comm, s));
    return CP_OK;
  }
  CP_NCCL(ncclGroupStart());
  for (int r = 0; r < g.n; ++r) {
    const size_t cnt = (size_t)(g.start[r + 1] - g.start[r]);
    if (cnt == 0) continue;
    ncclResult_t rr = ncclBroadcast(buf + g.start[r], buf + g.start[r], cnt, ncclFloat, r, c->comm, s);
    if (rr != ncclSuccess) {
      ncclGroupEnd();
      CP_FAIL(CP_ERR_NCCL, std::string("ncclBroadcast: ") + ncclGetErrorString(rr));
    }
  }
  CP_NCCL(ncclGroupEnd());
  return CP_OK;
}

int comm_sum_blocks(cp_comm c, float* buf, const Blocks& g, int dx_mode, cudaStream_t s) {
  if (!c || c->world == 1 || dx_mode == CP_DX_LOCAL) return CP_OK;
  if (c->loop) CP_FAIL(CP_ERR_UNSUPPORTED, "loopback communicator: NCCL collectives unavailable (fused paths only)");
  CP_TRY(async_error(c));
  if (dx_mode == CP_DX_ALLREDUCE) {
    CP_NCCL(ncclAllReduce(buf, buf, (size_t)g.start[g.n], ncclFloat, ncclSum, c->comm, s));
    return CP_OK;
  }
  if (equal_widths(g)) {
    const size_t cnt = (size_t)(g.start[1] - g.start[0]);
    if (cnt == 0) return CP_OK;
    CP_NCCL(ncclReduceScatter(buf, buf + g.start[c->rank], cnt, ncclFloat, ncclSum, c->comm, s));
    return CP_OK;
  }
  CP_NCCL(ncclGroupStart());
  for (int r = 0; r < g.n; ++r) {
    const size_t cnt = (size_t)(g.start[r + 1] - g.start[r]);
    if (cnt == 0) continue;
    ncclResult_t rr = ncclReduce(buf + g.start[r], buf + g.start[r], cnt, ncclFloat, ncclSum, r, c->comm, s);
    if (rr != ncclSuccess) {
      ncclGroupEnd();
      CP_FAIL(CP_ERR_NCCL, std::string("ncclReduce: ") + ncclGetErrorString(rr));
    }
  }
  CP_NCCL(ncclGroupEnd());
  return CP_OK;
}

}  // namespace cp
