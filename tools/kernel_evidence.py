"""Per-kernel roofline evidence from one `ncu --set full` capture of a frame
(no GPU needed): duration, achieved DRAM bandwidth vs the measured peak,
shared-memory wavefront and L2 atomic throughput as % of their peaks, issue
rate (warp instructions per SM cycle vs 4) and achieved occupancy.

  python tools/kernel_evidence.py gpurun_out/frame_end.ncu-rep > profiles/r1_kernel_evidence.md
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "nsecond": 1e-9, "msecond": 1e-3}
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs", 6536.0))

    def val(d, k):
        v = d.get(k, "")
        try:
            return float(v.replace(",", "")) * scale.get(units[hdr.index(k)], 1.0)
        except (ValueError, KeyError):
            return float("nan")

    print(f"# Per-kernel evidence ({os.path.basename(rep)}, one config-2 frame, ncu cold-cache replays)\n")
    print("DRAM peak: measured %.0f GB/s (MEASURED_PEAKS.json).  Shared-memory and L2-atomic columns are ncu's "
          "own `pct_of_peak_sustained_elapsed`; issue = warp instructions per SM per cycle (peak 4).\n" % hbm)
    print("| kernel | time (µs) | DRAM (MB) | DRAM GB/s (% peak) | smem wavefronts (% peak) | smem atomics (% peak) "
          "| L2 atomic unit busy / L1 atomic requests (% peak) | issue (IPC / 4) | warps active |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("ges::", "").replace("void ", "")
        t = val(d, "gpu__time_duration.sum")
        dram = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
        gbs = dram / t / 1e9
        sm_wf = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "nan")
        sm_at = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed", "nan")
        try:   # L2 atomic unit busy (avg over slices) and the global atomic requests issued by L1
            l2 = (f"{float(d['lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed']):.1f} / "
                  f"{float(d['l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum.pct_of_peak_sustained_elapsed']):.1f}")
        except (KeyError, ValueError):
            l2 = "n/a"
        ipc = d.get("sm__inst_executed.avg.per_cycle_active", "nan")
        occ = d.get("sm__warps_active.avg.pct_of_peak_sustained_active", "nan")
        print(f"| `{name}` | {t * 1e6:.1f} | {dram / 1e6:.1f} | {gbs:.0f} ({100 * gbs / hbm:.0f} %) | "
              f"{float(sm_wf):.1f} % | {float(sm_at):.1f} % | {l2} | {float(ipc):.2f} ({25 * float(ipc):.0f} %) | "
              f"{float(occ):.0f} % |")


if __name__ == "__main__":
    main(sys.argv[1])
