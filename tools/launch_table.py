"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) of the last forward in the log:
python tools/launch_table.py gpurun_out/launches.csv [n_last_launches]"""
import csv, collections, sys

def load(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    ix = {h: j for j, h in enumerate(hdr)}
    launches = collections.OrderedDict()
    for r in rows[i + 1:]:
        key = (r[0], r[ix["Kernel Name"]])
        launches.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    return list(launches.items())

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}

def val(m, k):
    if k not in m:
        return 0.0
    v, u = m[k]
    return float(v.replace(",", "")) * SCALE.get(u, 1.0)

if __name__ == "__main__":
    items = load(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else len(items)
    items = items[-n:]
    agg = collections.OrderedDict()
    for (_, name), m in items:
        k = name.split("(")[0].replace("void ", "")[:48]
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += val(m, "gpu__time_duration.sum")
        a[2] += val(m, "dram__bytes_read.sum") + val(m, "dram__bytes_write.sum")
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':48s} {'n':>4s} {'us total':>10s} {'us/launch':>10s} {'share':>6s} {'GB/s':>7s}")
    for k, (c, t, b) in agg.items():
        print(f"{k:48s} {c:4d} {t:10.1f} {t / c:10.2f} {t / tot:6.3f} {b / t / 1e3 if t else 0:7.0f}")
    print(f"total {tot:.1f} us over {len(items)} launches")
