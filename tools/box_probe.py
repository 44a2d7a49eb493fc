"""Box facts for the offload denominators: host topology and
pinned cudaMemcpyAsync bandwidth D2H / H2D / bidirectional at 16 MiB..1 GiB.
Writes JSON to gpurun_out/box_probe.json."""

import json
import os
import subprocess
import time

import torch


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=30).stdout
    except Exception as e:  # pragma: no cover
        return str(e)


def bw(nbytes, direction, reps=5):
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    host2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dev2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if direction in ("d2h", "bidir"):
            with torch.cuda.stream(s1):
                host.copy_(dev, non_blocking=True)
        if direction in ("h2d", "bidir"):
            with torch.cuda.stream(s2):
                dev2.copy_(host2, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        moved = nbytes * (2 if direction == "bidir" else 1)
        best = max(best, moved / dt / 1e9)
    return best


def main():
    out = {"lscpu": sh("lscpu | head -20"), "topo": sh("nvidia-smi topo -m"), "numa": sh("numactl -H 2>/dev/null | head"),
           "affinity": len(os.sched_getaffinity(0)), "gpu": torch.cuda.get_device_name(0), "pinned_gbs": {}}
    for mib in (16, 64, 256, 1024):
        n = mib << 20
        out["pinned_gbs"][mib] = {d: round(bw(n, d), 2) for d in ("d2h", "h2d", "bidir")}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/box_probe.json", "w"), indent=1)
    print(json.dumps(out["pinned_gbs"]))


if __name__ == "__main__":
    main()
