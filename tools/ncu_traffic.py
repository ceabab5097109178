"""Summarise an `ncu --set full` capture of in-pipeline kernel launches into the
`traffic` figures bench.py reports (DRAM bytes per launch vs algorithmic bytes).

Capture (on the GPU box, one GPU; CE mode verifies per 512 MiB span, so launch 2 of
the first load is a full span, algorithmic bytes = 512 MiB read):

    ncu --set full --clock-control none --import-source on -k regex:materialise_tma \
        -s 2 -c 1 -o gpurun_out/prof_pipeline_ce \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-standalone

Summarise (here):

    python tools/ncu_traffic.py gpurun_out/prof_pipeline_ce.ncu-rep ce 536870912 \
        > profiles/r01/ncu_traffic_ce.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,"
           "sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,"
           "syslts__t_sectors_aperture_sysmem_lookup_miss.sum")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1, "nsecond": 1e-9}


def main():
    rep, mode, alg = sys.argv[1], sys.argv[2], int(sys.argv[3])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", METRICS],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    launches = []
    for r in data:
        d = {}
        for h, u, v in zip(head, units, r):
            if h in METRICS.split(","):
                d[h] = float(v.replace(",", "")) * (SCALE.get(u, 1) if u != "sector" else 1)
        d["kernel"] = r[head.index("Kernel Name")]
        launches.append(d)
    L = launches[0]
    traffic = L["dram__bytes_read.sum"] + L["dram__bytes_write.sum"]
    print(json.dumps({
        "mode": mode, "capture": rep.split("/")[-1], "kernel": L["kernel"],
        "grid": int(L["launch__grid_size"]), "algorithmic_bytes": alg,
        "dram_bytes": traffic, "dram_read": L["dram__bytes_read.sum"], "dram_write": L["dram__bytes_write.sum"],
        "traffic_over_algorithmic": traffic / alg, "duration_s": L["gpu__time_duration.sum"],
        "dram_pct_of_peak": L.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        # host (sysmem) sectors the kernel pulled through the L2 -- the PCIe reads of a zero-copy launch
        "sysmem_read_bytes": 32 * L.get("syslts__t_sectors_aperture_sysmem_lookup_miss.sum", 0.0),
        "sysmem_over_algorithmic": 32 * L.get("syslts__t_sectors_aperture_sysmem_lookup_miss.sum", 0.0) / alg,
        "note": "ncu replays the launch with caches flushed (cold), serialised: the duration is not the "
                "in-pipeline time; the byte counts are the kernel's DRAM traffic for that launch"}, indent=1))


if __name__ == "__main__":
    main()
