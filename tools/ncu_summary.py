"""Dev tool: compact text summaries of ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launch-list.csv>   per-kernel launch table
  python tools/ncu_summary.py full <report.ncu-rep>         key metrics of each captured kernel
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 (DFMA) inst % of peak"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA tensor subpipe inst % of peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (elapsed)"),
]


def launches(path):
    lines = open(path).read().splitlines()
    i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(lines[i:]))
    agg = collections.OrderedDict()
    for r in rows:
        k = (r["Kernel Name"].split("(")[0][:90], r["Grid Size"], r["Block Size"])
        agg.setdefault(k, collections.defaultdict(list))[r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
    tot = sum(sum(m.get("gpu__time_duration.sum", [0])) for m in agg.values())
    print(f"source: {path}\nkernel | grid | block | launches | avg us | share of listed time | avg DRAM MB read")
    for (name, g, b), m in agg.items():
        t = m.get("gpu__time_duration.sum", [0])
        dr = m.get("dram__bytes_read.sum")
        print(f"{name} | {g} | {b} | {len(t)} | {sum(t) / len(t) / 1e3:.1f} | {sum(t) / tot:.1%} | "
              + (f"{sum(dr) / len(dr) / 1e6:.1f}" if dr else "-"))


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    print(f"source: {path}")
    for v in rows[2:]:
        d = dict(zip(h, v))
        print(f"\n== {d.get('Kernel Name', '?')[:120]}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:32s} {d[k]} {units.get(k, '')}".rstrip())
        st = [(k, d[k]) for k in h if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("ratio")]
        st = sorted(((float(x.replace(",", "")), k) for k, x in st if x), reverse=True)[:5]
        print("  top stall reasons (warps per issue): " +
              ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                        f" {x:.2f}" for x, k in st))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
