"""Static SASS instruction counts of the product kernels in libsb200.so
(profiles/r01_sass_evidence.md).  Run here; needs only cuobjdump.

    python scripts/sass_counts.py > profiles/r01_sass_evidence.md
"""
import re
import subprocess
import sys

LIB = "paper_2009_10917_b200/lib/libsb200.so"
OPS = ["UBLKCP", "SYNCS", "LDG", "STG", "LDS", "STS", "SHFL", "DFMA", "DADD", "DMUL", "BAR.SYNC", "ATOM",
       "MEMBAR"]
KERNELS = [
    ("BS6 (p >= 4)", "k_bs6_lanes<128, 512, false, 10>"),
    ("BS6 (p = 1)", "k_bs6_pairs<128, 512, true, 12>"),
    ("BS7", "k_bs7_lanes<128, 4, false, false>"),
    ("BS5 (n >= 3e6)", "k_lattice_tma<256, 4, 2, 4, 1, 4>"),
    ("BS5 (small n)", "k_lattice<256, 1, 2, 4>"),
    ("BS4 (n >= 1.6e7)", "k_lattice_tma<256, 1, 1, 2, 4, 1>"),
    ("BS4 (small n)", "k_lattice<256, 1, 1, 8>"),
    ("BS3 (n >= 4.8e7)", "k_lattice_tma<256, 1, 0, 2, 8, 1>"),
    ("BS3 (small n)", "k_lattice<256, 1, 0, 16>"),
    ("BS2", "k_elem_vec<1, 4, 256, false>"),
    ("BS1", "k_elem_vec<0, 4, 256, false>"),
]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            funcs[cur] = []
            continue
        if cur is not None:
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                funcs[cur].append(m.group(1))
    w = sys.stdout.write
    w("# SASS evidence (round 1, `cuobjdump -sass paper_2009_10917_b200/lib/libsb200.so`)\n\n")
    w("Static instruction counts per product kernel (`scripts/sass_counts.py`).  `UBLKCP` = TMA bulk\n"
      "copy (`cp.async.bulk`), `SYNCS` = mbarrier operations; `DFMA` must be 0 in every streaming\n"
      "kernel (no contraction: bitwise numpy rounding; checked by\n"
      "`tests/test_host_logic.py::test_library_is_sm100a`).  The lattice kernels have no `ATOM`: CTA 0\n"
      "collects the other CTAs' block values from flagged 8-byte slots\n"
      "(`profiles/r01_lattice_latency.md`); their `MEMBAR.ALL.SYS` belongs to the NCCL LSA barrier of\n"
      "the multi-GPU combine, executed only with an LSA context.  No tensor-core instructions\n"
      "anywhere: nothing on this path is a contraction.\n\n")
    w("| test | kernel | " + " | ".join(OPS) + " |\n|---|---|" + "---|" * len(OPS) + "\n")
    for test, name in KERNELS:
        hits = [f for f in funcs if f.startswith("void sb::" + name + "(")]
        if not hits:
            w(f"| {test} | `{name}` | " + " | ".join("?" for _ in OPS) + " |\n")
            continue
        ins = funcs[hits[0]]
        counts = [sum(1 for i in ins if i == op or i.startswith(op + ".")) for op in OPS]
        w(f"| {test} | `{name}` | " + " | ".join(str(c) for c in counts) + " |\n")


if __name__ == "__main__":
    main()
