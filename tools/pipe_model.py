"""Model of the host-buffer forward (sffn_forward_host): a three-stage pipeline H2D -> compute -> D2H over row chunks,
2 X / 2 Y staging slots, compute chunks in order.  Per-row costs fitted to the CUPTI timeline of the 7B pipeline
(profiles/r02/e2e_timeline_7B.txt: a 4096-row chunk's H2D 650-680 us while D2H runs, compute ~690 us).
Prints the modelled e2e time of chunk plans and how the best plan moves with the per-chunk fixed compute cost.
Usage: python tools/pipe_model.py"""
import math

H_CONC, H_ALONE = 0.1635, 0.149  # us per row (bf16, K = 4096) with / without the other direction busy
M = 32768


def sim(plan, fixed=95.0, per_row=0.145, slots=2):
    n = len(plan)
    h_end, c_end, d_end = [0.0] * n, [0.0] * n, [0.0] * n
    t_h = t_c = t_d = 0.0
    for i, r in enumerate(plan):
        start = t_h if i < slots else max(t_h, c_end[i - slots])          # X slot free
        h_end[i] = t_h = start + r * (H_CONC if i > 0 else H_ALONE)
        cs = max(h_end[i], t_c, d_end[i - slots] if i >= slots else 0.0)  # Y slot free
        c_end[i] = t_c = cs + fixed + r * per_row
        d_end[i] = t_d = max(c_end[i], t_d) + r * (H_CONC if i < n - 1 else H_ALONE)
    return d_end[-1]


def best(fixed, per_row):
    res = []
    for first in (512, 1024, 2048, 4096):
        for mid in (2048, 3072, 4096, 6144, 8192):
            for last in (512, 1024, 2048, 4096):
                rest = M - first - last
                if rest <= 0:
                    continue
                k = math.ceil(rest / mid)
                each = rest // k
                plan = [first] + [each] * (k - 1) + [rest - each * (k - 1)] + [last]
                res.append((sim(plan, fixed, per_row), first, mid, last, len(plan)))
    return min(res)


if __name__ == "__main__":
    for name, plan in [("library default (4096, ramp 2048)", [2048] + [4096] * 7 + [2048]),
                       ("2048 everywhere", [2048] * 16),
                       ("8192 with ramp", [2048, 4096, 8192, 8192, 4096, 4096, 2048])]:
        print(f"{name:36s} {sim(plan):7.0f} us")
    for fixed in (95, 60, 30, 0):
        for pr in (0.145, 0.135):
            t, f, m, l, n = best(fixed, pr)
            print(f"fixed {fixed:3d} us + {pr} us/row: best {t:7.0f} us (first {f}, middle {m}, last {l}, {n} chunks)")
