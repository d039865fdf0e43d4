"""Summarise ncu CSV exports: launch list and key metrics of a --set full capture."""
import csv, sys

def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            print(f'{d["Kernel Name"][:70]:70s} {float(d["Metric Value"])/1e3:10.1f} us')

KEYS = ("Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "L2 Hit Rate", "L1/TEX Hit Rate", "Achieved Occupancy", "Registers Per Thread",
        "Memory Throughput", "SM Frequency", "Eligible Warps Per Scheduler", "No Eligible")

def details(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    seen = set()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = (d.get("ID"), d.get("Metric Name"))
        if d.get("Metric Name") in KEYS and k not in seen:
            seen.add(k)
            print(f'[{d.get("ID")}] {d.get("Kernel Name","")[:30]:30s} {d["Metric Name"]:32s} {d["Metric Value"]:>12s} {d["Metric Unit"]}')

def raw(path, metrics):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("--", d.get("Kernel Name", "")[:60])
        for m in metrics:
            for h in hdr:
                if h == m:
                    print(f"   {m:60s} {d[h]} {units[hdr.index(h)]}")

if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches": launches(path)
    elif mode == "details": details(path)
    else: raw(path, sys.argv[3:])
