"""Summarise an ncu --set full report of the seven BS kernels into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_r01f.ncu-rep r01 [launches.csv]

Writes profiles/<tag>_ncu_summary.md (one row per kernel: duration, DRAM
bytes, achieved vs algorithmic bytes, DRAM %, occupancy, top stalls) and
updates profiles/traffic.json (DRAM bytes per launch, read by bench.py).
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# order of launches in scripts/profile_kernels.py's captured pass
TESTS = ["bs1", "bs2", "bs3", "bs4", "bs5", "bs6", "bs7"]
KEYS = {"bs1": "k_elem_vec<0>", "bs2": "k_elem_vec<1>", "bs3": "k_lattice_tma<norm>",
        "bs4": "k_lattice_tma<dot>", "bs5": "k_lattice_tma<fused>", "bs6": "k_bs6_lanes",
        "bs7": "k_bs7_lanes"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v) * scale


def bs6_section(specs):
    """Extra rows: the BS6 product kernel at config 3's N=1/2 (scripts/profile_bs6_low.py)."""
    from paper_2009_10917_b200.core import bytes_moved
    out = ["", "BS6 at config 3's low orders (NG ~ 1e8; scripts/profile_bs6_low.py, the product path):", "",
           "| N | kernel | duration us | DRAM read GB | DRAM write GB | traffic / algorithmic | achieved GB/s "
           "(algorithmic) | DRAM % peak | L1 % peak | issue active % | regs | achieved occ % | top stalls |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for spec in specs:
        rep, p = spec.rsplit(":", 1)
        p = int(p)
        K = int(round((1e8 ** (1 / 3) - 1) / p))
        ng, nl = (K * p + 1) ** 3, K ** 3 * (p + 1) ** 3
        algo = bytes_moved("bs6", nl=nl, ng=ng)
        hdr, units, rows = raw(rep)
        col = {h: i for i, h in enumerate(hdr)}
        r = rows[-1]

        def get(name):
            i = col.get(name)
            return (r[i], units[i]) if i is not None else ("", "")
        dur_v, dur_u = get("gpu__time_duration.sum")
        dur_us = float(dur_v) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(dur_u, 1.0)
        rd = to_bytes(*get("dram__bytes_read.sum"))
        wr = to_bytes(*get("dram__bytes_write.sum"))
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        out.append(f"| {p} | `{get('Kernel Name')[0].split('(')[0]}` | {dur_us:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                   f"{(rd + wr) / algo:.3f} | {algo / (dur_us * 1e-6) / 1e9:.0f} | "
                   f"{float(get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')[0]):.1f} | "
                   f"{float(get('l1tex__throughput.avg.pct_of_peak_sustained_active')[0] or 'nan'):.1f} | "
                   f"{float(get('smsp__issue_active.avg.pct_of_peak_sustained_active')[0] or 'nan'):.1f} | "
                   f"{get('launch__registers_per_thread')[0]} | "
                   f"{float(get('sm__warps_active.avg.pct_of_peak_sustained_active')[0]):.1f} | "
                   + ", ".join(f"{s} {v:.1f}" for v, s in stalls[:3]) + " |")
    return out


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    extra = [sys.argv[i + 1] for i, a in enumerate(sys.argv) if a == "--bs6"]
    from paper_2009_10917_b200.core import bytes_moved
    n = 100_000_000
    nl, ng = 147197952, 99252847  # K=66, N=7
    algo = {t: bytes_moved(t, n=n) for t in TESTS[:5]}
    algo["bs6"] = bytes_moved("bs6", nl=nl, ng=ng)
    algo["bs7"] = bytes_moved("bs7", nl=nl, ng=ng)
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, name):
        i = col.get(name)
        return (r[i], units[i]) if i is not None else ("", "")

    lines = [f"# ncu --set full summary ({tag})", "",
             "Workload: scripts/profile_kernels.py (bench step: BS1-BS5 n=1e8, BS6/BS7 K=66 N=7), "
             "one captured launch per kernel, `--clock-control none`, cold L2 (ncu replays).", "",
             "| test | kernel | duration us | DRAM read GB | DRAM write GB | traffic / algorithmic | "
             "achieved GB/s (algorithmic) | DRAM % peak | L1 % peak | issue active % | regs | achieved occ % | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}

    def test_of(kname):
        if "k_elem_vec<0" in kname:
            return "bs1"
        if "k_elem_vec<1" in kname:
            return "bs2"
        if "k_lattice" in kname:
            mode = kname.split("<")[1].split(",")[2].strip()
            return {"0": "bs3", "1": "bs4", "2": "bs5"}[mode]
        if "k_bs6_" in kname:
            return "bs6"
        if "k_bs7" in kname:
            return "bs7"
        return None

    picked = {}
    for r in rows:
        t = test_of(get(r, "Kernel Name")[0])
        if t is not None:
            picked[t] = r  # the last (warm) launch of each kernel
    for t in TESTS:
        if t not in picked:
            continue
        r = picked[t]
        name = get(r, "Kernel Name")[0].split("(")[0]
        dur_v, dur_u = get(r, "gpu__time_duration.sum")
        dur_us = float(dur_v) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(dur_u, 1.0)
        rd = to_bytes(*get(r, "dram__bytes_read.sum"))
        wr = to_bytes(*get(r, "dram__bytes_write.sum"))
        pct = get(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")[0]
        regs = get(r, "launch__registers_per_thread")[0]
        l1 = get(r, "l1tex__throughput.avg.pct_of_peak_sustained_active")[0] or "nan"
        iss = get(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")[0] or "nan"
        occ = get(r, "sm__warps_active.avg.pct_of_peak_sustained_active")[0]
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        top = ", ".join(f"{s} {v:.1f}" for v, s in stalls[:3])
        ach = algo[t] / (dur_us * 1e-6) / 1e9
        lines.append(f"| {t} | `{name}` | {dur_us:.1f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                     f"{(rd + wr) / algo[t]:.3f} | {ach:.0f} | {float(pct):.1f} | {float(l1):.1f} | {float(iss):.1f} | {regs} | "
                     f"{float(occ):.1f} | {top} |")
        traffic[KEYS[t]] = int(rd + wr)
    if extra:
        lines += bs6_section(extra)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    path = os.path.join(ROOT, "profiles", "traffic.json")
    with open(path, "w") as f:
        json.dump({"source": f"profiles/{tag}_ncu_summary.md (ncu --set full, dram__bytes_read.sum + "
                             "dram__bytes_write.sum per launch)", **traffic}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
