"""Summarise ncu raw CSV exports and a launch list into profiles/<round>_ncu_summary.md.

usage: python tools/summarize_ncu.py <round> <launches.csv> <raw.csv>... > profiles/<round>_ncu_summary.md
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (%)", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (%)", 1),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (%)", 1),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1),
    ("lts__t_sectors.sum", "L2 sectors (M)", 1e-6),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)", 1),
    ("launch__registers_per_thread", "registers/thread", 1),
    ("launch__grid_size", "grid", 1),
]


def raw_rows(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        out.append((d, u))
    return out


def fnum(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    rnd, launches, raws = sys.argv[1], sys.argv[2], sys.argv[3:]
    print(f"# ncu summary — {rnd}\n")
    print("Captured with `ncu --metrics gpu__time_duration.sum --clock-control none` (launch list) and")
    print("`ncu --set full --clock-control none --import-source on -k regex:<kernels> -c N` (tools/gpu_round.sh), on")
    print("one B200, running `bench.py --steps 1 --no-graph` (C2 workload). ncu times are cold-cache and serialised: compare")
    print("shares, not absolutes. Units as reported by ncu (MB = 1e6 bytes unless ncu says otherwise).\n")
    rows = list(csv.reader(open(launches)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    # last step only (the final len(step) launches)
    names = [d["Kernel Name"] for d in data]
    start = max(i for i, n in enumerate(names) if "select_kernel" in n)
    step = data[start:]
    tot = sum(float(d["Metric Value"]) for d in step)
    print("## Launch list of one step (device time per launch)\n")
    print("| # | kernel | us | share |")
    print("|---|---|---|---|")
    for i, d in enumerate(step):
        t = float(d["Metric Value"]) / 1000
        print(f"| {i} | `{d['Kernel Name'][:70]}` | {t:.1f} | {100 * t * 1000 / tot:.1f}% |")
    print(f"\nTotal device time of the step's launches: {tot / 1000:.1f} us ({len(step)} launches).\n")
    print("## Per-kernel metrics (ncu --set full)\n")
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for path in raws:
        for d, u in raw_rows(path):
            vals = []
            for k, _, sc in KEYS:
                v = fnum(d.get(k))
                unit = u.get(k, "")
                if v is None:
                    vals.append("-")
                    continue
                if "bytes" in k:
                    mult = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3, "Tbyte": 1e6}.get(unit, 1)
                    v *= mult
                    vals.append(f"{v:.1f}")
                elif k == "lts__t_sectors.sum":
                    vals.append(f"{v * 1e-6:.1f}")
                elif k == "gpu__time_duration.sum":
                    mult = {"nsecond": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
                    vals.append(f"{v * mult:.1f}")
                else:
                    vals.append(f"{v:.1f}")
            name = d.get("Kernel Name", "?")[:60]
            print(f"| `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
