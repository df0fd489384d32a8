"""Validates the reference arm's extrapolation (bench.py StockReference): times the stock
prefillsim.numerics.block_forward_hybrid (baseline/_ref) for one Llama-3.1-8B-shaped layer at 1k/2k/4k tokens (the
bench's fit points) and then at 8,192 and 20,000 tokens, and compares the measured seconds with the fit's prediction.
python tools/ref_layer_check.py > profiles/r2_reference_fit_check.json (GPU box host; ~1 min of CPU)"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402

nm = bench._stock_numerics()
assert nm is not None, "baseline/_ref not installed"
ref = bench.StockReference(nm)
ref.step(512, record=False)
for n in (1024, 2048, 4096):  # the round-2 (first) fit points
    ref.step(n)
a, b = ref.fit()
out = {"fit_points": {n: t for n, t in ref.samples}, "fit": {"a_per_token": a, "b_per_token2": b}, "checks": {}}
for n in (8192, 20_000):
    t0 = time.perf_counter()
    dt = ref.step(n, record=False)
    pred = a * n + b * n * n
    out["checks"][n] = {"measured_s": dt, "predicted_s": pred, "ratio_measured_over_predicted": dt / pred}
out["host_cpus"] = os.cpu_count()
out["blas"] = bench.blas_name()
out["request_seconds_measured_layer_x32"] = 32 * out["checks"][20_000]["measured_s"]
out["tokens_per_s_from_measured_20k_layer"] = 20_000 / out["request_seconds_measured_layer_x32"]
print(json.dumps(out, indent=1))
