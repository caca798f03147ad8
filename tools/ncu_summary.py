"""Summarise ncu output into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv> <tag>
      -> profiles/launches_<tag>.md (+ .csv): the last forward step's
         launches with device time, share of the step and DRAM bytes, and
         profiles/traffic.json (per-step DRAM bytes of the grouped GEMMs).
  python tools/ncu_summary.py full <report.ncu-rep> <tag>
      -> profiles/ncu_full_<tag>.md: key metrics per captured kernel."""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"


def short(name: str) -> str:
    n = name.split("(")[0].replace("void ", "").replace("moe::", "")
    return n[:70]


TOKENS = 16384   # bench --tokens of the captured command (argv[4] overrides)


def launches(path: str, tag: str):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    by_id = OrderedDict()
    for r in rows:
        k = by_id.setdefault(int(r["ID"]), {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        k[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ks = list(by_id.values())
    # the last step: from the last router launch to the end
    start = max(i for i, k in enumerate(ks) if "router_gate" in k["name"] or "router_tc" in k["name"])
    step = ks[start:]
    tot = sum(k["gpu__time_duration.sum"] for k in step)
    out = [f"# Launch list, last forward step ({tag})", "",
           "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
           "(cold-cache, serialised: compare shares, not absolutes) of "
           "`python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e`.", "",
           f"Step total (sum of launches): {tot / 1e6:.3f} ms, {len(step)} launches.", "",
           "| # | kernel | grid | block | time (us) | share | DRAM read (MB) | DRAM write (MB) |",
           "|---|---|---|---|---|---|---|---|"]
    for i, k in enumerate(step):
        t = k["gpu__time_duration.sum"]
        out.append(f"| {i} | `{short(k['name'])}` | {k['grid']} | {k['block']} | {t / 1e3:.1f} | {t / tot * 100:.1f}% | "
                   f"{k.get('dram__bytes_read.sum', 0) / 1e6:.1f} | {k.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    (PROF / f"launches_{tag}.md").write_text("\n".join(out) + "\n")
    gem = [k for k in step if "gemm_i8_tc" in k["name"]]
    traffic = {"tag": tag, "tokens": TOKENS, "grouped_gemm_bytes_per_step": sum(k.get("dram__bytes_read.sum", 0) +
                                                                k.get("dram__bytes_write.sum", 0) for k in gem),
               "per_kernel": [{"kernel": short(k["name"]), "us": k["gpu__time_duration.sum"] / 1e3,
                               "dram_read": k.get("dram__bytes_read.sum", 0),
                               "dram_write": k.get("dram__bytes_write.sum", 0)} for k in step]}
    (PROF / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(out))


FULL_METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor mem active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
]


def full(path: str, tag: str):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = [f"# ncu --set full summary ({tag})", "", f"Report: `{Path(path).name}` (not committed; regenerate with "
           "the command in DESIGN.md §Measurement).", "",
           "| kernel | " + " | ".join(lbl for _, lbl in FULL_METRICS) + " |",
           "|---|" + "---|" * len(FULL_METRICS)]
    for r in data:
        cells = []
        for m, _ in FULL_METRICS:
            if m in h:
                i = h.index(m)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        out.append(f"| `{short(r[h.index('Kernel Name')])}` | " + " | ".join(cells) + " |")
    # top stall reasons (PC sampling) per kernel
    st_cols = [(i, c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, c in enumerate(h)
               if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
    out += ["", "Top warp stall reasons (PC sampling, share of samples):", ""]
    for r in data:
        vals = []
        for i, n in st_cols:
            try:
                vals.append((n, float(r[i].replace(",", ""))))
            except ValueError:
                pass
        tot = sum(v for _, v in vals) or 1.0
        top = ", ".join(f"{n} {v / tot * 100:.0f}%" for n, v in sorted(vals, key=lambda x: -x[1])[:5])
        out.append(f"- `{short(r[h.index('Kernel Name')])}`: {top}")
    (PROF / f"ncu_full_{tag}.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    mode, path, tag = sys.argv[1:4]
    if len(sys.argv) > 4:
        TOKENS = int(sys.argv[4])
    (launches if mode == "launches" else full)(path, tag)
