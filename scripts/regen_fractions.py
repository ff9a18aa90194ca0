"""Rewrite the round-1 fraction-of-peak columns against ONE denominator:
MEASURED_PEAKS.json hbm_gbs (driver-measured copy peak on this pool's B200s),
with the nominal 8 TB/s beside it.

    python scripts/regen_fractions.py profiles/r01_model_fit.md profiles/r01_bs6_variants.md
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
NOMINAL = 8000.0


def fix_table(lines, i):
    """lines[i] is a header row holding 'Wmax / 6650'; rewrite that column and add a nominal one."""
    hdr = [c.strip() for c in lines[i].strip().strip("|").split("|")]
    col = next(k for k, c in enumerate(hdr) if c.startswith("Wmax / 6650"))
    wcol = hdr.index("Wmax (GB/s)")
    hdr[col] = f"Wmax / {PEAK:.0f} (measured)"
    hdr.insert(col + 1, "/ 8000 (nominal)")
    out = ["| " + " | ".join(hdr) + " |"]
    sep = [c for c in lines[i + 1].strip().strip("|").split("|")]
    sep.insert(col + 1, "---")
    out.append("|" + "|".join(sep) + "|")
    j = i + 2
    while j < len(lines) and lines[j].startswith("|"):
        cells = [c.strip() for c in lines[j].strip().strip("|").split("|")]
        w = float(cells[wcol])
        cells[col] = f"{w / PEAK:.2f}"
        cells.insert(col + 1, f"{w / NOMINAL:.2f}")
        out.append("| " + " | ".join(cells) + " |")
        j += 1
    return out, j


def fix_row_table(lines, i):
    """A '| / 6650 |' row under a GB/s row (r01_bs6_variants.md)."""
    prev = [c.strip() for c in lines[i - 1].strip().strip("|").split("|")]
    vals = [f"{float(v) / PEAK:.2f}" for v in prev[1:]]
    nom = [f"{float(v) / NOMINAL:.2f}" for v in prev[1:]]
    return [f"| / {PEAK:.0f} (measured) | " + " | ".join(vals) + " |",
            "| / 8000 (nominal) | " + " | ".join(nom) + " |"], i + 1


def main(paths):
    for p in paths:
        lines = open(p).read().split("\n")
        out, i = [], 0
        while i < len(lines):
            ln = lines[i]
            if ln.startswith("|") and "Wmax / 6650" in ln:
                rows, i = fix_table(lines, i)
                out += rows
            elif ln.startswith("| / 6650 |"):
                rows, i = fix_row_table(lines, i)
                out += rows
            else:
                out.append(re.sub(r"of the 6650 GB/s fallback peak",
                                  f"of the {PEAK:.0f} GB/s measured peak", ln))
                i += 1
        open(p, "w").write("\n".join(out))
        print("rewrote", p)


if __name__ == "__main__":
    main(sys.argv[1:])
