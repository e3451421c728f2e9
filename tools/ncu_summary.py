"""Summarise ncu reports here (no GPU needed): per-kernel duration, DRAM bytes,
throughputs, occupancy, top stall reasons and the hottest SASS lines.

  python tools/ncu_summary.py gpurun_out/x.ncu-rep [--sass N] [--launches file.csv]
"""
import argparse
import csv
import io
import subprocess
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append((d, u))
    return out


def sass(rep, top):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    res = []
    i = 0
    while i < len(rows):
        if rows[i] and rows[i][0] == "Kernel Name":
            name = rows[i][1]
            hdr = rows[i + 1]
            j = i + 2
            data = []
            while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
                data.append(rows[j])
                j += 1
            ist = hdr.index("Warp Stall Sampling (All Samples)")
            iex = hdr.index("Instructions Executed")
            isrc = hdr.index("Source")
            stalls = defaultdict(int)
            for r in data:
                for k, c in enumerate(hdr):
                    if c.startswith("stall_") and "Not Issued" not in c and r[k]:
                        stalls[c] += int(r[k])
            hot = sorted(((int(r[ist] or 0), int(r[iex] or 0), n, r[isrc].strip()) for n, r in enumerate(data)),
                         reverse=True)[:top]
            res.append((name, sorted(stalls.items(), key=lambda kv: -kv[1])[:8], sorted(hot, key=lambda t: t[2])))
            i = j
        else:
            i += 1
    return res


def lines(rep, kernel_regex, top):
    """Per CUDA source line: warp-level instructions executed and stall samples."""
    out = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kernel_regex}")
    rows = list(csv.reader(io.StringIO(out)))
    agg = []
    cur_file = None
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("Function Name",) or not r[0]:
            continue
        try:
            ex = int(r[hdr.index("Instructions Executed")] or 0)
            st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        agg.append((ex, st, f"{cur_file}:{r[0]}", r[1].strip()[:80]))
    tot_ex = sum(a[0] for a in agg) or 1
    tot_st = sum(a[1] for a in agg) or 1
    print(f"total warp-instructions {tot_ex}, stall samples {tot_st}")
    for ex, st, loc, src in sorted(agg, key=lambda a: -a[0])[:top]:
        print(f"  {ex / tot_ex:6.1%} inst {st / tot_st:6.1%} stall  {loc:22s} {src}")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        d[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print(f"{'kernel':70s} {'n':>4s} {'mean_us':>9s} {'share':>6s}")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:70]:70s} {len(v):4d} {sum(v) / len(v) / 1e3:9.1f} {sum(v) / tot:6.1%}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", nargs="?")
    ap.add_argument("--sass", type=int, default=0)
    ap.add_argument("--launches")
    ap.add_argument("--lines", help="kernel regex: per-source-line breakdown")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--traffic-json", help="write per-frame DRAM bytes and warp instructions (bench roofline input)")
    ap.add_argument("--b-alg", type=float, default=340272000.0)
    a = ap.parse_args()
    if a.traffic_json:
        import json
        dram, inst = {}, {}
        for d, u in raw(a.rep):
            name = d.get("Kernel Name", "?").split("(")[0].replace("ges::", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = sum(float(d[k].replace(",", "")) * scale.get(u.get(k, "byte"), 1)
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            dram[name] = dram.get(name, 0.0) + b
            inst[name] = inst.get(name, 0.0) + float(d["smsp__inst_executed.sum"].replace(",", ""))
        out = {"config": 2, "source": f"{a.rep} (ncu --set full, one frame, cold-cache replay)",
               "dram_bytes_per_frame": sum(dram.values()), "per_kernel": dram,
               "b_alg_bytes_per_frame": a.b_alg, "warp_instructions_per_frame": sum(inst.values()),
               "warp_instructions_per_kernel": inst}
        with open(a.traffic_json, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out, indent=1))
    if a.launches:
        launches(a.launches)
    if a.lines:
        lines(a.rep, a.lines, a.top)
        return
    if a.rep:
        for d, u in raw(a.rep):
            print("==", d.get("Kernel Name", "?")[:100])
            for k in KEYS:
                if k in d:
                    print(f"   {k:70s} {d[k]:>14s} {u.get(k, '')}")
        if a.sass:
            for name, stalls, hot in sass(a.rep, a.sass):
                print("== SASS", name[:80])
                print("   stalls:", ", ".join(f"{k[6:]}={v}" for k, v in stalls))
                for st, ex, n, src in hot:
                    print(f"   {n:5d} stall={st:6d} exec={ex:10d} {src[:90]}")


if __name__ == "__main__":
    main()
