"""Key metrics of every kernel in an `ncu --set full` report (read with ncu -i ... --page raw --csv).

python tools/ncu_full_summary.py gpurun_out/x.ncu-rep | gpurun_out/x_raw.csv
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
]


def main(rep):
    if rep.endswith(".csv"):  # raw page already exported on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    cols = [(k, n) for k, n in WANT if k in idx]
    print("| kernel | grid x block | " + " | ".join(n for _, n in cols) + " |")
    print("|---" * (len(cols) + 2) + "|")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0]
        gb = f'{r[idx["Grid Size"]]} x {r[idx["Block Size"]]}'
        vals = [f"{r[idx[k]]} {units[idx[k]]}".strip() for k, _ in cols]
        print(f"| `{name}` | {gb} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
