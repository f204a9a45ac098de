"""Host<->device copy bandwidth into pinned buffers allocated under each
NUMA node's CPU affinity (the e2e read-back of 4.3 GB of fields ran at
5.8 GB/s on one box and 54 GB/s on others).  Tuning aid.

    python tools/pcie_probe.py
"""
import json
import os
import time

import torch


def nodes():
    base = "/sys/devices/system/node"
    out = {}
    for d in sorted(os.listdir(base)) if os.path.isdir(base) else []:
        if d.startswith("node") and d[4:].isdigit():
            with open(os.path.join(base, d, "cpulist")) as fh:
                txt = fh.read().strip()
            cpus = set()
            for part in txt.split(","):
                if "-" in part:
                    a, b = part.split("-")
                    cpus.update(range(int(a), int(b) + 1))
                elif part:
                    cpus.add(int(part))
            if cpus:
                out[int(d[4:])] = sorted(cpus)
    return out


def bw(host, dev):
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("h2d", lambda: dev.copy_(host, non_blocking=True)),
                     ("d2h", lambda: host.copy_(dev, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name] = round(3 * host.numel() * host.element_size() / (time.perf_counter() - t0) / 1e9, 1)
    return res


def main():
    torch.cuda.set_device(0)
    n = (1 << 30) // 8
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    everyone = os.sched_getaffinity(0)
    out = {"cpus": len(everyone), "nodes": {}}
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, 4)
        local = [64 * w + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1]
        out["gpu_local_cpus"] = [min(local), max(local), len(local)] if local else None
    except Exception as exc:  # pragma: no cover
        out["gpu_local_cpus"] = repr(exc)
    host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out["default"] = bw(host, dev)
    del host
    for node, cpus in nodes().items():
        os.sched_setaffinity(0, set(cpus) & everyone or everyone)
        host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        host.fill_(1.0)
        out["nodes"][node] = {"cpus": [cpus[0], cpus[-1]], **bw(host, dev)}
        del host
    os.sched_setaffinity(0, everyone)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
