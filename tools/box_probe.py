"""Box facts for the offload denominators (SURVEY §7 step 1, §8(e) "the real
coupling is the host link"): host topology, each GPU's NUMA node, and pinned
cudaMemcpyAsync bandwidth D2H / H2D / bidirectional at 16 MiB..1 GiB — for every
visible GPU alone AND for all visible GPUs copying at the same time (the 8-GPU
case where every rank offloads through shared PCIe switches and host DRAM).
Host buffers come from sppo_host_alloc (NUMA-local to each GPU).
Writes JSON to gpurun_out/box_probe.json."""

import json
import os
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=30).stdout
    except Exception as e:  # pragma: no cover
        return str(e)


class Rig:
    """Per-GPU buffers: device src/dst and NUMA-local pinned host buffers."""

    def __init__(self, dev, nbytes):
        from paper_2503_10377_b200 import sppo
        torch.cuda.set_device(dev)
        self.dev = dev
        self.ctx = sppo.Context(dev)
        self.n = nbytes
        self.d1 = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
        self.d2 = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
        self.h1, self.h2 = self.ctx.host_alloc(nbytes), self.ctx.host_alloc(nbytes)
        self.numa = self.ctx.numa_node()

    def run(self, direction):
        """One copy (or one each way) through the ABI's copy streams; returns bytes moved."""
        torch.cuda.set_device(self.dev)
        s = torch.cuda.current_stream(self.dev)
        if direction in ("d2h", "bidir"):
            self.ctx.kv_offload(0, self.d1, self.h1, self.n, 1.0, producer=s)
        if direction in ("h2d", "bidir"):
            self.ctx.kv_prefetch(0, self.h2, self.d2, self.n, consumer=s, flags=1)
        self.ctx.sync()
        return self.n * (2 if direction == "bidir" else 1)

    def close(self):
        self.ctx.host_free(self.h1)
        self.ctx.host_free(self.h2)
        self.ctx.close()


def measure(rigs, direction, reps=5):
    """Aggregate GB/s with all `rigs` copying at once (threads, one per GPU); best of reps."""
    best = 0.0
    for _ in range(reps):
        bar = threading.Barrier(len(rigs) + 1)
        moved = [0] * len(rigs)

        def work(k):
            bar.wait()
            moved[k] = rigs[k].run(direction)

        th = [threading.Thread(target=work, args=(k,)) for k in range(len(rigs))]
        for t in th:
            t.start()
        bar.wait()
        t0 = time.perf_counter()
        for t in th:
            t.join()
        dt = time.perf_counter() - t0
        best = max(best, sum(moved) / dt / 1e9)
    return best


def main():
    n_gpu = torch.cuda.device_count()
    out = {"lscpu": sh("lscpu | head -20"), "topo": sh("nvidia-smi topo -m"), "numa": sh("numactl -H 2>/dev/null | head"),
           "affinity": len(os.sched_getaffinity(0)), "gpu": torch.cuda.get_device_name(0), "gpus": n_gpu,
           "pinned_gbs": {}, "concurrent_gbs": {}, "numa_nodes": []}
    for mib in (16, 64, 256, 1024):
        n = mib << 20
        rigs = [Rig(g, n) for g in range(n_gpu)]
        out["numa_nodes"] = [r.numa for r in rigs]
        out["pinned_gbs"][mib] = {d: round(measure(rigs[:1], d), 2) for d in ("d2h", "h2d", "bidir")}
        agg = {d: round(measure(rigs, d), 2) for d in ("d2h", "h2d", "bidir")}
        out["concurrent_gbs"][mib] = {"gpus": n_gpu, "aggregate": agg,
                                      "per_gpu": {d: round(v / n_gpu, 2) for d, v in agg.items()}}
        for r in rigs:
            r.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/box_probe.json", "w"), indent=1)
    print(json.dumps({"alone": out["pinned_gbs"], "concurrent": out["concurrent_gbs"], "numa": out["numa_nodes"]}))


if __name__ == "__main__":
    main()
