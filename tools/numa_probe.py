"""Host-link bandwidth vs NUMA placement of the pinned buffer (run under gpurun).
Prints the GPU's PCI-local CPU list and, for each NUMA node, the pinned H2D
cudaMemcpy rate and the zero-copy random-row gather rate with the allocating
thread bound to that node."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402


def node_cpus():
    out = {}
    for p in sorted(glob.glob("/sys/devices/system/node/node*/cpulist")):
        node = int(p.split("node")[-1].split("/")[0])
        out[node] = open(p).read().strip()
    return out


def parse(lst):
    s = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-")
            s.update(range(int(a), int(b) + 1))
        elif part:
            s.add(int(part))
    return s


props = torch.cuda.get_device_properties(0)
bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
info = {"gpu_pci": bus, "nodes": node_cpus()}
try:
    info["gpu_numa_node"] = open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip()
    info["gpu_local_cpus"] = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
except OSError as e:
    info["err"] = str(e)
print(json.dumps(info), flush=True)

from paper_2112_08541_b200 import _lib  # noqa: E402

nbytes = 256 << 20
dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
for node, cl in node_cpus().items():
    os.sched_setaffinity(0, parse(cl))
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    best = 0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dst.copy_(src, non_blocking=True)
        e.record()
        e.synchronize()
        best = max(best, nbytes / (s.elapsed_time(e) * 1e-3) / 1e9)
    # zero-copy gather of 100k random 400-B rows from this buffer
    rows = nbytes // 400
    ids = torch.randint(0, rows, (100000,), dtype=torch.int32, device="cuda").sort().values
    pos = torch.arange(100000, dtype=torch.int32, device="cuda")
    cnt = torch.tensor([100000], dtype=torch.int64, device="cuda")
    out = torch.empty((100000, 400), dtype=torch.uint8, device="cuda")
    tab = _lib.host_device_pointer(src)
    res = {}
    for ctas in (74, 148):
        for _ in range(2):
            _lib.call("bgl_gather_list", pos.data_ptr(), cnt.data_ptr(), 100000, ids.data_ptr(), tab, 400,
                      out.data_ptr(), None, None, 2, ctas, _lib.stream_ptr())
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5):
            _lib.call("bgl_gather_list", pos.data_ptr(), cnt.data_ptr(), 100000, ids.data_ptr(), tab, 400,
                      out.data_ptr(), None, None, 2, ctas, _lib.stream_ptr())
        e.record()
        e.synchronize()
        res[ctas] = round(5 * 100000 * 400 / (s.elapsed_time(e) * 1e-3) / 1e9, 2)
    print(json.dumps({"node": node, "memcpy_h2d_gbs": round(best, 2), "zero_copy_gather_gbs": res}), flush=True)
    del src
