"""Per-kernel SASS instruction summary of libirkb200.so (cuobjdump -sass).

usage: python tools/sass_summary.py [path/to/libirkb200.so] > profiles/<tag>_sass_summary.md
Counts the mnemonics that show which hardware path a kernel uses: DMMA (FP64
tensor core), UBLKCP (cp.async.bulk, the 1D TMA form), SYNCS (mbarrier),
LDG/STG/LDS/STS, DFMA, BAR, and the total instruction count.
"""
import collections
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["DMMA", "UBLKCP", "SYNCS", "DFMA", "DMUL", "DADD", "LDG", "STG", "LDS", "STS", "BAR", "SHFL", "REDUX",
        "ACQBULK", "UTMALDG", "UTCMMA"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "paper_1701_07181_b200", "csrc", "libirkb200.so")
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    dem = {}
    cur = None
    counts = collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
        if m:
            op = m.group(1)
            counts[cur]["total"] += 1
            for k in KEYS:
                if op.startswith(k):
                    counts[cur][k] += 1
    names = list(counts)
    if names:
        d = subprocess.run(["c++filt"] + names, capture_output=True, text=True).stdout.splitlines()
        dem = dict(zip(names, d))
    print("# SASS instruction summary (sm_100a), `cuobjdump -sass libirkb200.so`\n")
    print("Counts are static instructions per kernel. DMMA = FP64 tensor-core MMA (mma.sync.m8n8k4.f64; tcgen05 has no")
    print("f64 kind), UBLKCP = cp.async.bulk (1D TMA), SYNCS = mbarrier arrive/try_wait.\n")
    print("| kernel | total | " + " | ".join(KEYS[:13]) + " |")
    print("|---|---|" + "---|" * 13)
    tot = collections.Counter()
    for n in names:
        c = counts[n]
        tot.update(c)
        short = re.sub(r"\(.*$", "", dem.get(n, n)).replace("void ", "")
        print(f"| `{short}` | {c['total']} | " + " | ".join(str(c[k]) for k in KEYS[:13]) + " |")
    print(f"| **all {len(names)} kernels** | {tot['total']} | " + " | ".join(str(tot[k]) for k in KEYS[:13]) + " |")
    print(f"\nUTMALDG (tensor-map TMA): {tot['UTMALDG']}, UTCMMA (tcgen05.mma): {tot['UTCMMA']} -- none expected: the blocks are")
    print("contiguous (1D bulk copies) and the arithmetic is FP64.")


if __name__ == "__main__":
    main()
