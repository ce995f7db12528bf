"""Summarise `ncu --page raw --csv` exports: one line per captured launch with the
metrics the profiles/ summaries quote (duration, DRAM bytes, DRAM and tensor-pipe
utilisation, SM throughput, registers, grid, block, SM clock).

usage: python tools/ncu_summary.py OUT.txt RAW.csv [RAW.csv ...] [--traffic-json OUT.json]
       [--title "..."]

With --traffic-json the tc_gemm launches' dram__bytes_read.sum + dram__bytes_write.sum
(per launch, bytes) are written as the JSON bench.py reads for roofline.traffic.
"""
import argparse
import csv
import json

COLS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "clk"),
]

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,  # -> us
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,  # -> MB
         "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}  # -> GHz


def rows_of(path):
    with open(path) as f:
        r = list(csv.reader(f))
    hdr, units = r[0], r[1]
    out = []
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")}
        for key, _ in COLS:
            v = d.get(key)
            if v in (None, ""):
                rec[key] = None
                continue
            x = float(v.replace(",", ""))
            rec[key] = x * SCALE.get(u.get(key, ""), 1.0)
        out.append(rec)
    return out


def short(name):
    name = name.replace("void ", "").replace("c3d::", "").replace("(anonymous namespace)::", "")
    return name.split("(")[0][:58]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("raw", nargs="+")
    ap.add_argument("--traffic-json", default=None)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    recs = [r for p in a.raw for r in rows_of(p)]
    lines = []
    if a.title:
        lines.append("# " + a.title)
    lines.append("# columns: kernel, " + ", ".join(
        f"{k} [{'us' if 'time' in k else 'MB' if 'bytes' in k else 'GHz' if 'per_second' in k else ''}]"
        for k, _ in COLS))
    for r in recs:
        vals = []
        for key, _ in COLS:
            v = r[key]
            vals.append("-" if v is None else (f"{v:.0f}" if key.startswith("launch__") else f"{v:.3f}"))
        lines.append(f"{short(r['kernel']):58s}  " + "  ".join(vals))
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if a.traffic_json:
        per = [((r["dram__bytes_read.sum"] or 0) + (r["dram__bytes_write.sum"] or 0)) * 1e6
               for r in recs if "tc_gemm" in r["kernel"]]
        with open(a.traffic_json, "w") as f:
            json.dump({"bytes_per_launch": sum(per) / len(per) if per else None,
                       "launches": len(per), "per_launch_bytes": per,
                       "source": "ncu --set full --clock-control none of every tc_gemm launch of "
                                 "one cfg3 N=1 layer step (tools/profile_step.py 1): "
                                 "dram__bytes_read.sum + dram__bytes_write.sum; summary in "
                                 + a.out}, f, indent=1)


if __name__ == "__main__":
    main()
