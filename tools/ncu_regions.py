"""Source-page analysis of an ncu --set full --import-source on capture (tooling).

  ncu -i rep.ncu-rep --page source --csv --kernel-name regex:NAME --print-source sass > src.csv
  python tools/ncu_regions.py regions src.csv [header_row]
      splits the kernel's SASS at barriers / mbarrier waits / hot branches and prints, per
      region, its share of the stall samples, of the executed instructions, the FP64 share
      and the top stall reasons
  python tools/ncu_regions.py util src.csv header_row kernel_cycles lo:hi:name [lo:hi:name ...]
      per address range (hex, last 5 digits): time share, shared-memory wavefronts per SM
      against the 1 wavefront/clk/SM rate, IPC per SMSP, FP64 pipe utilisation (2 clk / warp instr)
  python tools/ncu_regions.py list src.csv header_row lo hi
      the instructions of a range with samples, executions and their two top stall reasons
header_row = 0-based index of the CSV row holding the column names of the wanted kernel
(a capture with several launches concatenates them).
"""
import collections
import csv
import re
import sys

FP64 = ("DFMA", "DMUL", "DADD", "DSETP")


def load(path, start):
    rows = list(csv.reader(open(path)))
    hdr = rows[start]
    ix = {k: i for i, k in enumerate(hdr)}
    data = []
    for r in rows[start + 1:]:
        if not r or r[0] == "Kernel Name":
            break
        data.append(r)
    return hdr, ix, data


def opcode(src):
    return re.sub(r"^@!?U?P\d+\s+", "", src).split()[0]


def regions(path, start):
    hdr, ix, data = load(path, start)
    f = lambda r, k: float(r[ix[k]] or 0)  # noqa: E731
    stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    tot = sum(f(r, "# Samples") for r in data)
    toti = sum(f(r, "Instructions Executed") for r in data)
    print("total samples", tot, "instructions", toti)
    cur = None

    def flush(a, why):
        nonlocal cur
        if cur and (cur["s"] > 0 or cur["i"] > 0):
            top = ", ".join("%s=%.1f%%" % (k[6:], 100 * v / tot) for k, v in cur["st"].most_common(5))
            print("%s..%s  samp %5.1f%%  inst %5.1f%% fp64 %4.1f%%  [%s]  end:%s" % (
                cur["a0"], a, 100 * cur["s"] / tot, 100 * cur["i"] / toti, 100 * cur["d"] / toti, top, why))
        cur = None

    for r in data:
        a, src = r[0][-5:], r[1]
        if cur is None:
            cur = {"s": 0, "i": 0, "d": 0, "st": collections.Counter(), "a0": a}
        cur["s"] += f(r, "# Samples")
        cur["i"] += f(r, "Instructions Executed")
        op = opcode(src)
        if op.split(".")[0] in FP64:
            cur["d"] += f(r, "Instructions Executed")
        for k in stalls:
            cur["st"][k] += f(r, k)
        hot_branch = (op.startswith("BRA") and ".U.ANY" not in src and f(r, "# Samples") > 0.002 * tot)
        if op.startswith("BAR") or "SYNCS.PHASECHK" in src or hot_branch or op.startswith("EXIT"):
            flush(a, src[:50])
    flush("end", "end")


def util(path, start, cycles, ranges):
    hdr, ix, data = load(path, start)
    f = lambda r, k: float(r[ix[k]] or 0)  # noqa: E731
    tot = sum(f(r, "# Samples") for r in data)
    rng = [(int(a, 16), int(b, 16), n) for a, b, n in (x.split(":") for x in ranges)]
    acc = {n: [0.0] * 5 for _, _, n in rng}
    for r in data:
        a = int(r[0][-5:], 16)
        for lo, hi, n in rng:
            if lo <= a <= hi:
                acc[n][0] += f(r, "# Samples")
                acc[n][1] += f(r, "L1 Wavefronts Shared")
                acc[n][2] += f(r, "L1 Wavefronts Shared Ideal")
                acc[n][3] += f(r, "Instructions Executed")
                if opcode(r[1]).split(".")[0] in FP64:
                    acc[n][4] += f(r, "Instructions Executed")
    for n, (s, w, wi, i, d) in acc.items():
        cyc = s / tot * cycles
        print("%-22s time %5.1f%%  cycles/SM %.3gM  smem wavefronts/SM %.3gM (ideal %.3gM) -> smem util %5.1f%%; "
              "instr/SMSP %.3gM IPC %.2f; FP64/SMSP %.3gM pipe %4.1f%%" % (
                  n, 100 * s / tot, cyc / 1e6, w / 148 / 1e6, wi / 148 / 1e6, 100 * w / 148 / max(cyc, 1),
                  i / 592 / 1e6, i / 592 / max(cyc, 1), d / 592 / 1e6, 200 * d / 592 / max(cyc, 1)))


def listing(path, start, lo, hi):
    hdr, ix, data = load(path, start)
    f = lambda r, k: float(r[ix[k]] or 0)  # noqa: E731
    stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    for r in data:
        a = int(r[0][-5:], 16)
        if lo <= a <= hi:
            st = sorted(((f(r, k), k[6:]) for k in stalls), reverse=True)[:2]
            print("%05x %-52s s%6.0f e%9.0f t%4.1f wf%9.0f %s" % (
                a, r[1][:52], f(r, "# Samples"), f(r, "Instructions Executed"), f(r, "Avg. Threads Executed"),
                f(r, "L1 Wavefronts Shared"), " ".join("%s:%.0f" % (k, v) for v, k in st if v > 0)))


if __name__ == "__main__":
    cmd, path = sys.argv[1], sys.argv[2]
    start = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    if cmd == "regions":
        regions(path, start)
    elif cmd == "util":
        util(path, start, float(sys.argv[4]), sys.argv[5:])
    else:
        listing(path, start, int(sys.argv[4], 16), int(sys.argv[5], 16))
