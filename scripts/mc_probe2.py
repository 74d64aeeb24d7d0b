"""2-rank probe: fabric-handle export/import of device memory and of a multicast object; multicast bind +
map; a multimem store from rank 0 visible on both ranks (via a tiny torch kernel? -> use cuMemcpy)."""
import os, sys, ctypes
import torch, torch.distributed as dist
from cuda.bindings import driver as cu
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
torch.cuda.synchronize()
def ck(r, what):
    err = r[0] if isinstance(r, tuple) else r
    print(f"[{rank}] {what}: {err}", flush=True)
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None
err, dev = cu.cuDeviceGet(rank)
for ht_name in ("CU_MEM_HANDLE_TYPE_FABRIC", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR"):
    ht = getattr(cu.CUmemAllocationHandleType, ht_name)
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = rank
    prop.requestedHandleTypes = ht
    size = 2 << 20
    h = ck(cu.cuMemCreate(size, prop, 0), f"{ht_name} cuMemCreate")
    if h is None: continue
    r = cu.cuMemExportToShareableHandle(h, ht, 0)
    print(f"[{rank}] {ht_name} export: {r[0]}", flush=True)
    mp = cu.CUmulticastObjectProp()
    mp.numDevices = world
    mp.handleTypes = ht
    mp.size = size
    if rank == 0:
        r2 = cu.cuMulticastCreate(mp)
        print(f"[{rank}] {ht_name} mc create: {r2[0]}", flush=True)
        if r2[0] == 0:
            r3 = cu.cuMemExportToShareableHandle(r2[1], ht, 0)
            print(f"[{rank}] {ht_name} mc export: {r3[0]}", flush=True)
            if ht_name.endswith("FABRIC") and r3[0] == 0:
                data = bytes(r3[1].data)
            else:
                data = (os.getpid(), int(r3[1]) if r3[0] == 0 else -1)
        else:
            data = None
    else:
        data = None
    obj = [data]
    dist.broadcast_object_list(obj, src=0)
    data = obj[0]
    if data is None: continue
    if rank != 0:
        if ht_name.endswith("FABRIC"):
            fh = cu.CUmemFabricHandle()
            fh.data = data
            r4 = cu.cuMemImportFromShareableHandle(fh, ht)
        else:
            pid, fd = data
            pidfd = os.pidfd_open(pid)
            try:
                myfd = int(ctypes.CDLL(None, use_errno=True).syscall(438, pidfd, fd, 0))
            except Exception as e:
                myfd = -1
            print(f"[{rank}] pidfd_getfd -> {myfd} errno {ctypes.get_errno()}", flush=True)
            r4 = cu.cuMemImportFromShareableHandle(myfd, ht) if myfd >= 0 else (-1, None)
        print(f"[{rank}] {ht_name} mc import: {r4[0]}", flush=True)
        mc = r4[1]
    else:
        mc = r2[1]
    if mc is not None:
        print(f"[{rank}] add device: {cu.cuMulticastAddDevice(mc, dev)[0]}", flush=True)
        dist.barrier()
        print(f"[{rank}] bind mem: {cu.cuMulticastBindMem(mc, 0, h, 0, size, 0)[0]}", flush=True)
        dist.barrier()
dist.destroy_process_group()
