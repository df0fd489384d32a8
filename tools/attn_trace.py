"""Per-tile pipeline timeline of one attention CTA from a -DATTN_TRACE build (clock64 stamps, SM cycles).

  tools/build_variant.sh trace attention.cu "-DATTN_TRACE=0"
  PREFILLONLY_LIB=build/variants/lib_trace.so python tools/attn_trace.py [n]

Events (see attention.cu TR()): slot i softmax: 4i wait-start, 4i+1 S ready, 4i+2 first half of P stored,
4i+3 P stored; MMA warp: 8/11 saw p_half of slot 0/1, 9/12 saw p_full, 10 saw next K tile, 13 issued S1(j+1);
loader: 14 stage free for tile j; 15/16/17 after issuing PV0 lo / PV0 hi / S0, 18/19 after PV1 lo / hi.
"""
import ctypes
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2505_07203_b200 import _lib  # noqa: E402

EV, TILES = 24, 512


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    hq, hkv = 32, 8
    ld = (hq + 2 * hkv) * 128
    qkv = torch.randn(n, ld, device="cuda").to(torch.bfloat16)
    out = torch.empty(n, hq * 128, dtype=torch.bfloat16, device="cuda")
    lib = _lib.load()
    for _ in range(3):
        _lib.call("po_op_attention", ctypes.c_void_p(qkv.data_ptr()), ld, n, 0, hq, hkv,
                  ctypes.c_void_p(out.data_ptr()), hq * 128, None)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (EV * TILES))()
    assert lib.po_debug_attn_trace(buf, EV * TILES) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(EV, TILES).astype(np.int64)
    nt = (n + 127) // 128
    lo, hi = 8, nt - 8
    t0 = t[1, 0]

    def med(x):
        return float(statistics.median(x))

    js = range(lo, hi)
    rep = {"n": n, "tiles": nt, "kernel_cycles_traced": int(t[3, nt - 1] - t0)}
    for i in (0, 1):
        w, r, h, e = t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]
        rep[f"slot{i}"] = {
            "period": med([r[j + 1] - r[j] for j in js]),
            "softmax_total(r->e)": med([e[j] - r[j] for j in js]),
            "softmax_first_half(r->h)": med([h[j] - r[j] for j in js]),
            "softmax_second_half(h->e)": med([e[j] - h[j] for j in js]),
            "wait_for_S(w->r)": med([r[j] - w[j] for j in js]),
            "P_done_to_next_S(e->r')": med([r[j + 1] - e[j] for j in js]),
        }
    rep["mma"] = {
        "p_half0 seen after arrive": med([t[8, j] - t[2, j] for j in js]),
        "p_full0 seen after arrive": med([t[9, j] - t[3, j] for j in js]),
        "k_full(j+1) seen after p_full0": med([t[10, j] - t[9, j] for j in js]),
        "p_half1 seen after arrive": med([t[11, j] - t[6, j] for j in js]),
        "p_full1 seen after arrive": med([t[12, j] - t[7, j] for j in js]),
        "slot1 S ready after S1 issue": med([t[5, j + 1] - t[13, j] for j in js]),
        "slot0 S ready after S0 issue(k seen)": med([t[1, j + 1] - t[10, j] for j in js]),
        "loader stage free(j+2) - k_full seen(j+1)": med([t[14, j + 2] - t[10, j] for j in range(lo, hi - 2)]),
    }
    rep["issue_cycles"] = {
        "PV0 lo": med([t[15, j] - t[8, j] for j in js]), "PV0 hi": med([t[16, j] - t[9, j] for j in js]),
        "S0": med([t[17, j] - t[10, j] for j in js]),
        "PV1 lo": med([t[18, j] - t[11, j] for j in js]), "PV1 hi": med([t[19, j] - t[12, j] for j in js]),
        "S1(+commit)": med([t[13, j] - t[19, j] for j in js]),
        "wait p_half0 (after S1 issued j-1)": med([t[8, j] - t[13, j - 1] for j in js]),
        "wait p_full0 (after PV0 lo)": med([t[9, j] - t[15, j] for j in js]),
        "wait k (after PV0 hi)": med([t[10, j] - t[16, j] for j in js]),
        "wait p_half1 (after S0)": med([t[11, j] - t[17, j] for j in js]),
        "wait p_full1 (after PV1 lo)": med([t[12, j] - t[18, j] for j in js]),
    }
    names = {0: "sm0 wait", 1: "sm0 S ready", 2: "sm0 P half", 3: "sm0 P done", 4: "sm1 wait", 5: "sm1 S ready",
             6: "sm1 P half", 7: "sm1 P done", 8: "mma saw p_half0", 9: "mma saw p_full0", 10: "mma saw K(j+1)",
             11: "mma saw p_half1", 12: "mma saw p_full1", 13: "mma issued S1(j+1)", 14: "ld K(j) stage free",
             15: "mma issued PV0 lo", 16: "mma issued PV0 hi", 17: "mma issued S0(j+1)", 18: "mma issued PV1 lo",
             19: "mma issued PV1 hi", 20: "ld V(j) stage free"}
    jr = nt // 2
    seq = sorted((int(t[e, j] - t[1, jr]), f"{names[e]} [{j}]") for e in names for j in (jr, jr + 1) if t[e, j])
    rep["raw_tile"] = [f"{c:6d} {nm}" for c, nm in seq if -3000 < c < 8000]
    rep["overlap_slot_softmax"] = med([max(0, min(t[3, j], t[7, j]) - max(t[1, j], t[5, j])) for j in js])
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
