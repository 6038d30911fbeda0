"""SASS evidence for the instruction claims in DESIGN.md §4/§7a (developer tool).

    python tools/sass_summary.py [lib.so] > profiles/r02/sass_summary.md

Runs `cuobjdump -sass` on the built library and tabulates, per kernel, the mnemonics that
prove a design choice: UBLKCP (cp.async.bulk = TMA bulk copy), SYNCS (mbarrier), DMMA
(fp64 tensor-core MMA), LDGSTS (cp.async), 128/256-bit vector loads, the L1::no_allocate
(.NA) and L2 eviction-hinted (.EF/.EL) streams, REDG/ATOMG (global reductions), VOTE/SHFL
(warp reductions).
"""
import collections
import re
import subprocess
import sys

KEYS = ["UBLKCP", "SYNCS", "DMMA", "LDGSTS", "LDG.*128", "LDG.*256", "LDG.E.NA", "EFL2", "REDG", "ATOMG", "VOTE",
        "SHFL", "LDS", "BAR.SYNC"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2212_10432_b200/libalphasparse.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None or "/*" not in line:
            continue
        ins = line.split("*/", 1)[1] if line.strip().startswith("/*") else line
        op = ins.strip().split(";")[0]
        if not op:
            continue
        funcs[cur]["n"] += 1
        for k in KEYS:
            if re.search(r"\b" + k, op):
                funcs[cur][k] += 1
    demangled = {}
    names = list(funcs)
    dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    for a, b in zip(names, dm):
        demangled[a] = b
    print(f"# SASS summary of `{lib}` (cuobjdump -sass, sm_100a)\n")
    print(f"{len(funcs)} kernels.  Totals over all kernels:\n")
    tot = collections.Counter()
    for c in funcs.values():
        tot.update(c)
    print("| " + " | ".join(["instructions"] + KEYS) + " |")
    print("|" + "---|" * (len(KEYS) + 1))
    print("| " + " | ".join([str(tot["n"])] + [str(tot[k]) for k in KEYS]) + " |\n")
    print("Kernels that carry a TMA / tensor-core / cp.async instruction, and one instantiation per family:\n")
    print("| kernel | " + " | ".join(["instructions"] + KEYS) + " |")
    print("|---|" + "---|" * (len(KEYS) + 1))
    seen = set()
    for f, c in funcs.items():
        nm = demangled[f]
        fam = re.sub(r"<.*", "", nm.replace("(anonymous namespace)::", ""))
        special = c["UBLKCP"] or c["DMMA"] or c["LDGSTS"]
        if not special and fam in seen:
            continue
        seen.add(fam)
        short = nm.replace("(anonymous namespace)::", "")
        short = re.sub(r"\(.*", "", short)
        print(f"| `{short}` | " + " | ".join([str(c["n"])] + [str(c[k]) for k in KEYS]) + " |")


if __name__ == "__main__":
    main()
