"""Summarise ncu captures into committed text (run here, no GPU needed).

    python profiles/summarize.py <tag> <launches.csv> <full.ncu-rep> [<more.ncu-rep> ...]

Writes profiles/<tag>_launches.txt (per-kernel share of the launch list:
cold-cache, serialised per-launch times — compare shares, not absolutes),
profiles/<tag>_ncu_full.txt (per-kernel key counters from `--set full`) and
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-inst"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-inst"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        t[name] += v * scale
        n[name] += 1
    tot = sum(t.values())
    out = ["kernel                                   launches   total_us   share"]
    for k, v in sorted(t.items(), key=lambda kv: -kv[1]):
        out.append(f"{k[:40]:40s} {n[k]:8d} {v:10.1f} {100 * v / tot:6.1f}%")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out, traffic, seen = [], {}, set()
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("hbgpu::", "").replace("void ", "")
        if name in seen:  # one capture per kernel
            continue
        seen.add(name)
        out.append(f"== {name}")
        for key, label in KEYS:
            if key in hdr:
                out.append(f"   {label:24s} {r[hdr.index(key)]:>16s} {units[hdr.index(key)]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        out.append("   top stalls (warps per issue): " + ", ".join(f"{s}={v:.2f}" for v, s in stalls[:6]))

        def val(key):
            v = float(r[hdr.index(key)])
            u = units[hdr.index(key)]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

        traffic.setdefault(name.split("<")[0], val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
    return "\n".join(out), traffic


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    with open(os.path.join(HERE, f"{tag}_launches.txt"), "w") as f:
        f.write(launches(lcsv) + "\n")
    text, traffic = "", {}
    for rep in reps:
        t, tr = full(rep)
        text += t + "\n"
        for k, v in tr.items():
            traffic.setdefault(k, v)
    text = text.rstrip("\n")
    with open(os.path.join(HERE, f"{tag}_ncu_full.txt"), "w") as f:
        f.write(text + "\n")
    with open(os.path.join(HERE, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print(open(os.path.join(HERE, f"{tag}_launches.txt")).read())
    print(text)


if __name__ == "__main__":
    main()
