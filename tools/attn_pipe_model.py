"""Discrete-event model of the attention CTA pipeline (one MMA issuer, in-order tensor pipe whose issue blocks at
execution rate, two softmax slots), calibrated on tools/attn_trace.py measurements. Used to choose the MMA issue
order and S/P layout before writing kernel code.

  python tools/attn_pipe_model.py
"""
import itertools

LAT_SEEN = 120      # barrier arrive -> MMA thread sees it
LAT_READY = 100     # MMA group complete -> softmax sees s_full
PV_HALF, S_FULL = 256, 512


def simulate(order, ts_half1, ts_half2, tiles=60, split_s=False):
    """order: 'static' (PV0, S0', PV1, S1' - the current kernel) or 'dynamic' (issue whichever slot's next
    group is ready first). split_s: S(j+1) issued as two N=64 halves; the half that does not overlap P(j) goes as
    soon as the softmax has read S(j) into registers. Returns cycles per tile (both slots)."""
    pipe_free = 0.0
    thread_t = 0.0
    s_ready = {(i, 0): (i + 1) * S_FULL + LAT_READY for i in (0, 1)}  # S0, S1 of tile 0 issued back to back
    pipe_free = 2 * S_FULL
    thread_t = pipe_free - 64
    sm_free = {0: 0.0, 1: 0.0}
    events = {}

    def softmax(i, j):
        start = max(s_ready[(i, j)], sm_free[i])
        h = start + ts_half1
        e = h + ts_half2
        sm_free[i] = e
        events[(i, j)] = (start + 120, h, e)   # +120: LDTM of S done (S buffer free for split_s)

    for i in (0, 1):
        softmax(i, 0)

    def issue(dep_time, dur):
        nonlocal pipe_free, thread_t
        start = max(dep_time + LAT_SEEN, thread_t, pipe_free)
        pipe_free = start + dur
        thread_t = pipe_free - 64
        return pipe_free

    nxt = {0: 0, 1: 0}
    done_tiles = 0
    while min(nxt.values()) < tiles - 1:
        if order == "static":
            seq = [0, 1]
        else:  # dynamic: the slot whose P(j) is ready first
            seq = sorted((0, 1), key=lambda i: events[(i, nxt[i])][1])
        for i in seq:
            j = nxt[i]
            _, h, e = events[(i, j)]
            if split_s:
                # S_hi(j+1) into the columns P(j) does not use: ready once S(j) was read
                t_hi = issue(events[(i, j)][0], S_FULL // 2)
                issue(h, PV_HALF)
                issue(e, PV_HALF)
                t_lo = issue(0, S_FULL // 2)
                s_ready[(i, j + 1)] = max(t_hi, t_lo) + LAT_READY
            else:
                issue(h, PV_HALF)
                issue(e, PV_HALF)
                s_ready[(i, j + 1)] = issue(0, S_FULL) + LAT_READY
            nxt[i] = j + 1
            softmax(i, j + 1)
        done_tiles += 1
    t_end = max(sm_free.values())
    return t_end / tiles


if __name__ == "__main__":
    print("measured: period 3268-3582 cycles/tile, softmax 880 + 630")
    for ts in [(880, 630), (700, 500), (600, 400), (500, 300)]:
        for order, split in itertools.product(("static", "dynamic"), (False, True)):
            p = simulate(order, *ts, split_s=split)
            print(f"softmax {ts} order={order:7s} split_s={split!s:5s}: {p:7.0f} cyc/tile  tensor {2048 / p:5.1%}")
