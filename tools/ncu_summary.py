"""Key numbers of an `ncu --page raw --csv` export (one launch): time, clock,
tensor / MUFU / smem pipe utilisation, DRAM and L2 bytes.
usage: python tools/ncu_summary.py prof_bwd_raw.csv [flops]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, val = rows[0], rows[1], rows[2]
d = dict(zip(hdr, val))
u = dict(zip(hdr, units))


def get(name):
    for h in hdr:
        if h == name:
            return float(d[h].replace(",", "")), u[h]
    return None, None


out = {}
for key, name in [("time", "gpu__time_duration.sum"), ("sm_clock", "sm__cycles_elapsed.avg.per_second"),
                  ("grid", "launch__grid_size"), ("cluster_x", "launch__cluster_dim_x"),
                  ("tensor_active_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                  ("tensor_mem_active_pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                  ("xu_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                  ("smem_tc_wavefront_pct", "l1tex__data_pipe_tc_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed"),
                  ("smem_lsu_wavefront_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed"),
                  ("dram_read", "dram__bytes_read.sum"), ("dram_write", "dram__bytes_write.sum"),
                  ("l2_red_pct", "lts__t_sectors_op_red.avg.pct_of_peak_sustained_elapsed"),
                  ("l2_throughput_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed")]:
    v, unit = get(name)
    if v is not None:
        out[key] = (v, unit)
for k, (v, unit) in out.items():
    print(f"{k:24s} {v:14.4f} {unit}")
if len(sys.argv) > 2 and "time" in out:
    t, unit = out["time"]
    t_s = t * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}[unit]
    print(f"{'tflops':24s} {float(sys.argv[2]) / t_s / 1e12:14.2f}")
