"""Opcode / pipe mix of the innermost hot loops of one kernel in an object or library.

    python tools/sass_loop.py build/obj/tl_aot.o 'k_aotILNS_7AotModeE0ELi6' [--min-ldg 4] [--show]

Finds backward branches (loops), keeps those whose body holds at least
--min-ldg global loads and no inner loop, and prints per loop: instruction
count, ALU-pipe / FMA-pipe / LSU / other split (B200: both integer pipes
issue one warp instruction per 2 cycles per SM sub-partition, the scheduler
one per cycle -- DESIGN §4, tools/pipe_bench.cu).  CPU-only (cuobjdump).
"""
import re
import subprocess
import sys
from collections import Counter

ALU = ("LOP3", "SHF", "IADD3", "ISETP", "VIADDMNMX", "VIMNMX", "VIMNMX3", "SEL", "LEA", "PRMT", "MOV", "VIADD", "IADD",
       "LOP", "BMSK", "SGXT", "IABS", "FMNMX", "PLOP3", "P2R", "R2P", "VOTE", "ICMP", "FSEL", "CS2R")
FMA = ("IMAD", "FFMA", "FMUL", "FADD", "HFMA2")
LSU = ("LDG", "LDS", "STS", "STG", "LDL", "STL", "ATOMS", "ATOMG", "RED", "LDGSTS", "LDSM", "ATOM")
XU = ("POPC", "FLO", "BREV", "MUFU", "I2F", "F2I")


def pipe(op):
    base = op.split(".")[0]
    if base in FMA:
        return "fma"
    if base in LSU:
        return "lsu"
    if base in XU:
        return "xu"
    if base in ALU:
        return "alu"
    if base.startswith("U") or base in ("S2UR", "R2UR", "LDCU"):
        return "uniform"
    return "other"


def kernel_sass(path, pattern):
    txt = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    out, on = [], False
    for line in txt.splitlines():
        if "Function :" in line:
            on = pattern in line
        elif on:
            m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
            if m:
                out.append((int(m.group(1), 16), m.group(2).strip()))
    return out


def main():
    path, pattern = sys.argv[1], sys.argv[2]
    min_ldg = int(sys.argv[sys.argv.index("--min-ldg") + 1]) if "--min-ldg" in sys.argv else 4
    show = "--show" in sys.argv
    ins = kernel_sass(path, pattern)
    addr_ix = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"\bBRA(?:\.\w+)*\s+(?:\w+,\s*)?0x([0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt <= a and tgt in addr_ix:
                loops.append((addr_ix[tgt], i))
    inner = [(s, e) for (s, e) in loops if not any((s2 > s or e2 < e) and s2 >= s and e2 <= e for (s2, e2) in loops if (s2, e2) != (s, e))]
    print(f"{len(ins)} instructions, {len(loops)} loops, {len(inner)} innermost")
    for s, e in inner:
        body = ins[s:e + 1]
        ops = [re.sub(r"^@!?U?P\d+\s+", "", t).split()[0] for _, t in body]
        nldg = sum(o.startswith("LDG") for o in ops)
        if nldg < min_ldg:
            continue
        pc = Counter(pipe(o) for o in ops)
        print(f"loop {ins[s][0]:#x}-{ins[e][0]:#x}: {len(body)} instr, LDG {nldg}, LDS {sum(o.startswith('LDS') for o in ops)} | " +
              " ".join(f"{k}={v}" for k, v in sorted(pc.items())))
        print("   ", dict(Counter(o.split('.')[0] for o in ops).most_common()))
        if show:
            for a, t in body:
                print(f"      {a:#06x}  {t}")


if __name__ == "__main__":
    main()
