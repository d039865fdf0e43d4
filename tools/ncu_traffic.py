"""Write profiles/ncu_traffic.json (per-kernel DRAM bytes per launch) from an `ncu --page raw --csv` export of
one sparse forward step (tools/prof_step.sh), plus a markdown table of the step's kernels."""
import csv, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SC = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}
NAMES = [("gemm_tc_kernel<0", "gate_gemm_twell"), ("union_rank", "union_rank"), ("permute_rows", "permute_rows"),
         ("union_meta", "union_meta"), ("union_gate_list", "union_gate_list"),
         ("union_gemm_kernel<1", "union_up_gemm"), ("union_gemm_kernel<0", "union_down_gemm")]
KEYS = {"t": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
        "tc": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "l2hit": "lts__t_sector_hit_rate.pct",
        "l2": "lts__throughput.avg.pct_of_peak_sustained_elapsed"}


def main(raw, cfg="7B", out=os.path.join(ROOT, "profiles", "ncu_traffic.json")):
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = next((n for pat, n in NAMES if pat in d["Kernel Name"]), None)
        if name is None:
            continue
        v = {}
        for k, m in KEYS.items():
            i = hdr.index(m)
            v[k] = float(d[m].replace(",", "")) * SC.get(units[i], 1.0)
        res[name] = v
    traffic = {n: int(v["rd"] + v["wr"]) for n, v in res.items()}
    doc = {"_source": "ncu --set full --clock-control none of one sffn_forward (tools/prof_step.sh), "
                      f"{cfg} config; dram__bytes_read.sum + dram__bytes_write.sum per launch",
           cfg: traffic}
    old = json.load(open(out)) if os.path.exists(out) else {}
    for k, v in old.get(cfg, {}).items():
        doc[cfg].setdefault(k, v)
    json.dump(doc, open(out, "w"), indent=2)
    print("| kernel | ncu time (ms) | DRAM read (GB) | DRAM write (GB) | tensor pipe % | L2 hit % | L2 throughput % |")
    print("|---|---|---|---|---|---|---|")
    for n, v in res.items():
        print(f"| {n} | {v['t']*1e3:.3f} | {v['rd']/1e9:.3f} | {v['wr']/1e9:.3f} | {v['tc']:.1f} | {v['l2hit']:.1f} | {v['l2']:.1f} |")
    print(f"| step total | {sum(v['t'] for v in res.values())*1e3:.3f} | {sum(v['rd'] for v in res.values())/1e9:.3f} | "
          f"{sum(v['wr'] for v in res.values())/1e9:.3f} | | | |")


if __name__ == "__main__":
    main(*sys.argv[1:])
