"""H2D bandwidth vs the NUMA placement of the pinned source (GPU-local cores vs the rest)."""
import json
import os
import subprocess

import torch

torch.cuda.init()
props = torch.cuda.get_device_properties(0)
bus = "%04x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
info = {"bus": bus}
try:
    info["local_cpulist"] = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
    info["numa_node"] = open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip()
except OSError as e:
    info["sysfs_err"] = str(e)
info["affinity_default"] = len(os.sched_getaffinity(0))
info["lscpu"] = [l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                 if "NUMA" in l or "Socket" in l or "Model name" in l]


def parse(cl):
    out = set()
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def bw():
    x = torch.empty(10000 * 784, dtype=torch.float32).pin_memory()
    d = torch.empty_like(x, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(x, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            d.copy_(x, non_blocking=True)
        e1.record(s)
        s.synchronize()
    return 10 * x.numel() * 4 / (e0.elapsed_time(e1) * 1e-3) / 1e9


allc = os.sched_getaffinity(0)
info["default_GBps"] = bw()
if "local_cpulist" in info:
    local = parse(info["local_cpulist"]) & allc
    remote = allc - local
    if local:
        os.sched_setaffinity(0, local)
        info["local_GBps"] = bw()
    if remote:
        os.sched_setaffinity(0, remote)
        info["remote_GBps"] = bw()
print(json.dumps(info))
