"""Per-kernel SASS instruction summary of the built library (run in the
build container; cuobjdump needs no GPU):

    python tools/sass_summary.py > profiles/r02/sass_summary.md

Counts, per kernel, the instructions that prove which units a kernel uses:
tcgen05 MMA (UTCHMMA / UTCQMMA...), TMEM loads (LDTM) and alloc (UTCATOMSWS),
TMA (UTMALDG / UTMASTG), fp64 (DFMA / DADD / DMUL), global loads (LDG),
shared (LDS / STS), and the register count from the ELF resource usage.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2101_10994_b200", "libnglod_b200.so")
CLASSES = [("UTC*MMA", re.compile(r"\bUTC\w*MMA\b")), ("LDTM", re.compile(r"\bLDTM\b")),
           ("UTCATOMSWS/UTCBAR", re.compile(r"\bUTC(ATOMSWS|BAR)\b")), ("UTMA*", re.compile(r"\bUTMA\w+\b")),
           ("DFMA/DADD/DMUL", re.compile(r"\bD(FMA|ADD|MUL)\b")), ("FFMA", re.compile(r"\bFFMA\b")),
           ("LDG", re.compile(r"\bLDG\b")), ("LDS", re.compile(r"\bLDS\b")), ("STS", re.compile(r"\bSTS\b")),
           ("ATOM/RED", re.compile(r"\b(ATOM|ATOMG|RED|REDG)\b")), ("BAR", re.compile(r"\bBAR\b"))]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True, check=True).stdout
    regs = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+)", res):
        regs[m.group(1)] = int(m.group(2))
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur and re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
            for name, rx in CLASSES:
                if rx.search(line):
                    counts[cur][name] += 1
            counts[cur]["total"] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
    print("# SASS summary of libnglod_b200.so (sm_100a)\n")
    print("`python tools/sass_summary.py` (cuobjdump -sass / -res-usage). Instruction counts are static "
          "(per kernel body, not executed).\n")
    print("| kernel | regs | " + " | ".join(n for n, _ in CLASSES) + " | total |")
    print("|---|---|" + "---|" * (len(CLASSES) + 1))
    for (mangled, c), pretty in zip(counts.items(), demangle):
        short = pretty.split("(")[0].replace("ng::", "")
        if len(short) > 60:
            short = short[:57] + "..."
        print(f"| `{short}` | {regs.get(mangled, '')} | " + " | ".join(str(c.get(n, 0)) for n, _ in CLASSES)
              + f" | {c['total']} |")


if __name__ == "__main__":
    sys.exit(main())
