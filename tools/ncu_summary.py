"""Summarise an `ncu --set full` report (.ncu-rep) into a short text file for profiles/.

    python tools/ncu_summary.py report.ncu-rep > profiles/r01_<kernel>.txt
Prints, per profiled kernel: duration, grid/block, registers, shared memory, achieved IPC,
FP64 pipe and shared-memory utilisation, DRAM/L2 traffic (bytes per launch: the roofline's
`traffic`), and the warp-stall breakdown (PC sampling).
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("smsp__issue_active.avg.per_cycle_active", "issue active (per SMSP)"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "DMMA instructions"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA sub-pipe % of peak (active)"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_elapsed", "DMMA sub-pipe % of peak (elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (active)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM read bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print("no kernels in", path)
        return
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        print(f"== {d.get('Kernel Name', '?')}")
        for k, name in KEYS:
            if k in d:
                print(f"  {name:28s} {d[k]} {u.get(k, '')}")
        st = {k: float(v) for k, v in d.items()
              if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
        print("  warp stalls: " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
