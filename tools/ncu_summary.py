"""Summarise one kernel of an .ncu-rep (ncu --set full) as 'Section | Metric | value unit' lines plus the DRAM
bytes (dram__bytes_read/write.sum) used as `roofline.traffic`:

    python tools/ncu_summary.py gpurun_out/x.ncu-rep "header line" > profiles/<round>_<kernel>_ncu.txt
"""
import csv
import io
import subprocess
import sys


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    print(f"# {header}")
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    iS, iN, iU, iV = hdr.index("Section Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    iK = hdr.index("Kernel Name")
    print(f"# kernel: {rows[1][iK][:160]}")
    for r in rows[1:]:
        if r[iS] in ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Scheduler Statistics",
                     "Warp State Statistics", "Launch Statistics", "Occupancy", "Compute Workload Analysis"):
            print(f"{r[iS]} | {r[iN]} | {r[iV]} {r[iU]}".rstrip())
    rr = list(csv.reader(io.StringIO(raw)))
    h, u, v = rr[0], rr[1], rr[2]
    for w in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum",
              "sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"):
        if w in h:
            i = h.index(w)
            print(f"raw | {w} | {v[i]} {u[i]}")


if __name__ == "__main__":
    main()
