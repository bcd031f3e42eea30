import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29517")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import torch.distributed._symmetric_memory as symm_mem
print("mc supported:", getattr(symm_mem, "is_nvshmem_available", lambda: None)())
try:
    t = symm_mem.empty(1024, dtype=torch.float32, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("buffer_ptrs", h.buffer_ptrs, "multicast_ptr", h.multicast_ptr, "world", h.world_size)
    print([a for a in dir(h) if not a.startswith("_")])
except Exception as e:
    print("symm_mem error", repr(e))
import subprocess
print(subprocess.run(["nvidia-smi","-q"],capture_output=True,text=True).stdout.count("Fabric"))
print(subprocess.run(["bash","-c","nvidia-smi -q | grep -i -A3 fabric | head -20"],capture_output=True,text=True).stdout)
from cuda.bindings import driver as drv
drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
print("MULTICAST_SUPPORTED", drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
dist.destroy_process_group()
