"""Write profiles/traffic_config2.json from one `ncu --set full` capture of a
config-2 frame (no GPU needed): DRAM bytes and warp instructions per kernel
and per frame -- bench.py's `roofline.traffic` and `roofline.issue` inputs.

  python tools/traffic_json.py gpurun_out/r2_frame.ncu-rep > profiles/traffic_config2.json
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "": 1}
FRAME = ("k_surfel_prep", "k_gauss3_prep", "k_scan", "k_fill", "k_tile")


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]

    def val(d, k):
        return float(d[k].replace(",", "")) * SCALE.get(units[hdr.index(k)], 1.0)

    dram, inst = {}, {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        if not any(k in name for k in FRAME) or name in dram:   # first launch of each kernel = one frame
            continue
        dram[name] = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
        inst[name] = val(d, "smsp__inst_executed.sum")
    json.dump({"config": 2,
               "source": f"{rep} (ncu --set full, one frame, cold-cache replay)",
               "dram_bytes_per_frame": sum(dram.values()), "per_kernel": dram,
               "b_alg_bytes_per_frame": 340272000.0,
               "warp_instructions_per_frame": sum(inst.values()), "warp_instructions_per_kernel": inst},
              sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
