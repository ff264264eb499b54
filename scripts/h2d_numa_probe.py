"""Pinned host-to-device bandwidth for the C2 query batch (12.6 MiB) with the process on each
NUMA node's CPUs (the pinned buffer is first-touched there).  Diagnostic only."""
import glob
import os
import time

import torch


def h2d_gbs(nb, reps=30):
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    return nb * reps / (s.elapsed_time(e) / 1e3) / 1e9


def cpus(spec):
    out = []
    for part in spec.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += range(int(a), int(b) + 1)
        elif part:
            out.append(int(part))
    return out


def main():
    torch.cuda.init()
    p = torch.cuda.get_device_properties(0)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        gnode = open(f"/sys/bus/pci/devices/{bus}/numa_node").read().strip()
    except OSError:
        gnode = "?"
    print("gpu", bus, "numa_node", gnode, "nproc", os.cpu_count())
    nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
    allc = os.sched_getaffinity(0)
    print("default affinity", len(allc), "cpus:", {mb: round(h2d_gbs(int(mb * 2**20)), 1) for mb in (4, 12.6, 64)})
    for nd in nodes:
        cs = set(cpus(open(nd + "/cpulist").read())) & allc
        if not cs:
            continue
        os.sched_setaffinity(0, cs)
        print(os.path.basename(nd), len(cs), "cpus:", {mb: round(h2d_gbs(int(mb * 2**20)), 1) for mb in (4, 12.6, 64)})
    os.sched_setaffinity(0, allc)


if __name__ == "__main__":
    main()
