"""Opcode summary of the shipped library's SASS (cuobjdump -sass): per
kernel, the instruction count and the tensor / copy opcodes that show which
hardware paths it uses (DMMA = FP64 tensor pipe, LDGSTS = cp.async, UBLKCP =
TMA-unit bulk copy, UTMALDG = tensor-map TMA, UTC*MMA = tcgen05).
python tools/sass_summary.py [lib.so] > profiles/<tag>_sass_summary.txt"""
import collections
import re
import subprocess
import sys

KEY = ("DMMA", "DFMA", "DMUL", "LDGSTS", "UBLKCP", "UTMALDG", "UTCMMA", "UTCHMMA", "LDS", "STS",
       "SYNCS", "BAR", "HMMA")


def main(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    kern, counts = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Za-z0-9_.]+)?", line)
        if m and kern:
            counts[kern]["_total"] += 1
            op = m.group(1) + (m.group(2) or "")
            for k in KEY:
                if op.startswith(k):
                    counts[kern][op] += 1
    print(f"# cuobjdump -sass {lib}")
    for k, c in counts.items():
        if not any(o.startswith(("DMMA", "LDGSTS", "UBLKCP")) for o in c):
            continue
        dem = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        ops = ", ".join(f"{o} {n}" for o, n in sorted(c.items()) if o != "_total")
        print(f"{dem[:110]}\n    {c['_total']} instructions; {ops}")
    allops = collections.Counter()
    for c in counts.values():
        allops.update(c)
    print("library totals:", ", ".join(f"{o} {allops[o]}" for o in sorted(allops) if o != "_total"))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2305_05581_b200/lib/libsdmrg_b200.so")
