"""Summarise ncu output into profiles/: python tools/ncu_summary.py <launches.csv> [<full.ncu-rep>] > out.md

* launch list (gpu__time_duration.sum, --clock-control none): per-kernel count, mean/total time and
  share of the hdf kernels' time (torch fill kernels = the L2 flush, listed but not counted);
* full capture: per kernel the headline counters (duration, DRAM bytes, DRAM/FMA/issue utilisation,
  occupancy, registers, shared memory)."""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name):
    m = re.search(r"(k_\w+)", name)
    return m.group(1) if m else name.split("(")[0][:60]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    agg = collections.OrderedDict()
    for r in rows:
        k = short(r[4])
        v = float(r[14].replace(",", ""))
        agg.setdefault(k, []).append(v)
    hdf_tot = sum(sum(v) for k, v in agg.items() if k.startswith("k_"))
    print(f"## Launch list `{path.split('/')[-1]}` (ncu --metrics gpu__time_duration.sum --clock-control none)\n")
    print("| kernel | launches | mean us | total us | share of hdf kernel time |")
    print("|---|---|---|---|---|")
    for k, v in agg.items():
        share = f"{100 * sum(v) / hdf_tot:.1f}%" if k.startswith("k_") else "(L2 flush / torch)"
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e3:.1f} | {share} |")
    print()


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma inst %"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "hmma inst %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"## Full capture `{path.split('/')[-1]}` (ncu --set full --clock-control none)\n")
    names = [m for m, _ in METRICS if m in col]
    print("| kernel | " + " | ".join(f"{lab} ({units[col[m]]})" for m, lab in METRICS if m in col) + " |")
    print("|---|" + "---|" * len(names))
    for r in rows[2:]:
        k = short(r[col["Kernel Name"]])
        print(f"| {k} | " + " | ".join(r[col[m]] for m in names) + " |")
    print()


if __name__ == "__main__":
    if sys.argv[1] == "--full-only":
        full(sys.argv[2])
    else:
        launches(sys.argv[1])
        if len(sys.argv) > 2:
            full(sys.argv[2])
