#!/usr/bin/env python
"""Per-kernel SASS instruction summary of the built libdpcuda.so (cuobjdump
-sass): total instructions and the counts of the mnemonics that show the
Blackwell-native design -- bulk TMA copies (UBLKCP / UTMALDG), mbarrier
sync (SYNCS), packed fp32 (FFMA2 / FADD2 / FMUL2), 128-bit global stores
(STG.E.*128) and their cache hints, shared-memory traffic, warp votes.

    python tools/sass_summary.py > profiles/sass_r2.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2101_12127_b200", "lib", "libdpcuda.so")
KEYS = ["UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "FFMA2", "FADD2", "FMUL2", "FFMA", "PRMT", "I2F", "LDS", "STS",
        "VOTE", "MATCH", "REDUX", "ATOMG", "RED", "BAR", "SHFL"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
        return out.splitlines()
    except OSError:
        return names


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else SO
    text = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            op = m.group(1)
            c = kernels[cur]
            c["total"] += 1
            base = op.split(".")[0]
            c[base] += 1
            if base in ("LDG", "STG") and op != base:
                c[op] += 1
    names = demangle(list(kernels))
    print(f"# SASS summary of {os.path.relpath(so, ROOT)} (cuobjdump -sass, sm_100a); counts are static "
          f"instructions per kernel\n")
    for (mangled, c), name in zip(kernels.items(), names):
        short = re.sub(r"dpk::\(anonymous namespace\)::", "", name)
        short = re.sub(r"\(.*", "", short) if "pipeline_kernel" not in short else short.split("(")[0]
        hits = [f"{k}={c[k]}" for k in KEYS if "." not in k and c.get(k)]
        hits += [f"{op}={n}" for op, n in sorted(c.items()) if op.split(".")[0] in ("LDG", "STG") and "." in op]
        print(f"{short}\n    total={c['total']}  " + "  ".join(hits))


if __name__ == "__main__":
    main()
