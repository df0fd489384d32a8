"""Per-launch key metrics of ncu reports (--page raw --csv) as JSON lines: python tools/ncu_rep_table.py a.ncu-rep ..."""
import csv, io, json, subprocess, sys

KEYS = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct", "sm__cycles_elapsed.avg.per_second": "sm_hz",
        "launch__grid_size": "grid"}

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"report": rep.split("/")[-1], "kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, short in KEYS.items():
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                if short == "us" and units[hdr.index(k)].strip() == "nsecond":
                    v = v / 1e3
                elif short == "us" and units[hdr.index(k)].strip() == "msecond":
                    v = v * 1e3
                d[short] = v
        print(json.dumps(d))
