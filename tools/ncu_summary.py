"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/ (tracked evidence)."""
import csv, io, json, subprocess, sys, collections
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "gpurun_out"
P = ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
        "smsp__average_warp_latency_per_inst_issued.ratio", "lts__t_bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


summary = {}
traffic = {}
for rep, cls in [("attn_full", "attention"), ("gemm_gateup_full", "gemm_gate_up_silu"),
                 ("gemm_down_full", "gemm_down_resid")]:
    f = G / f"{rep}.ncu-rep"
    if not f.exists():
        continue
    r = raw(f)
    m = {k: r[k] for k in KEYS if k in r}
    summary[rep] = {k: f"{v} {u}" for k, (v, u) in m.items()}

    def to_bytes(key):
        v, u = r[key]
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return float(v.replace(",", "")) * mult

    traffic[cls] = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
(P / f"{tag}_ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
if traffic:
    (P / "ncu_traffic.json").write_text(json.dumps({
        "source": f"ncu --set full, one launch per kernel ({tag}): dram__bytes_read.sum + dram__bytes_write.sum",
        "shapes": {"attention": "20k tokens, 32 q / 8 kv heads (tools/bench_attn.py)",
                   "gemm_gate_up_silu": "8192 x 28672 x 4096 (tools/bench_gemm.py)",
                   "gemm_down_resid": "8192 x 4096 x 14336 (tools/bench_gemm.py)"},
        "dram_bytes_per_launch": traffic}, indent=1) + "\n")

# launch list: time share per kernel family over one bench step
L = G / "launches.csv"
if L.exists():
    rows = [r for r in csv.reader(open(L)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "").strip()
        agg[name][0] += float(r[14].replace(",", "")) / 1e6
        agg[name][1] += 1
    tot = sum(v[0] for k, v in agg.items() if "init_" not in k)
    lines = ["| kernel | launches | ms (ncu, serialised) | share of step |", "|---|---|---|---|"]
    for k, (ms, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if "init_" in k:
            continue
        lines.append(f"| `{k}` | {c} | {ms:.2f} | {ms / tot:.3f} |")
    (P / f"{tag}_launches_summary.md").write_text(
        "# ncu launch list (one bench step incl. warm-up launches; `--metrics gpu__time_duration.sum "
        "--clock-control none`)\n\nPer-launch times are cold-cache and serialised: compare shares, not "
        "absolutes.\n\n" + "\n".join(lines) + "\n")
print(json.dumps(summary, indent=1)[:3000])
print(traffic)
