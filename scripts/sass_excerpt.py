"""profiles/rNN_sass_switch_umma.txt: opcode counts and excerpts of the dominant kernel's SASS (cuobjdump of the built library).
    python scripts/sass_excerpt.py r02 [mangled-name-substring]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2603_11873_b200", "libadafuse_b200.so")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
want = sys.argv[2] if len(sys.argv) > 2 else "switch_umma_kernelILi4ELb1ELi4ELi3ELb0E"   # <NB=4, GEMV, CH=4, PC=3, no peers>: the headline bench's kernel

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, name = collections.OrderedDict(), None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        funcs[name] = []
    elif name and re.match(r"\s+/\*[0-9a-f]{4,6}\*/", line):
        funcs[name].append(line.rstrip())
key = next(k for k in funcs if want in k)
body = funcs[key]
ops = collections.Counter()
for l in body:
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", l)
    if m:
        ops[m.group(1)] += 1
SHOW = ("UTCHMMA", "LDTM", "UTCBAR", "UTCATOMSWS", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "ATOMG", "RED", "ELECT", "R2UR", "UIADD3")
out = [f"# cuobjdump -sass paper_2603_11873_b200/libadafuse_b200.so   (nvcc 12.9, -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo); scripts/sass_excerpt.py",
       f"# kernel: {key}",
       "# Opcodes that show the Blackwell paths: UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld (accumulators out of tensor memory),",
       "# UTCBAR = tcgen05.commit -> mbarrier, UTCATOMSWS = tcgen05.alloc, UTMALDG / UTMASTG = TMA tensor loads / stores of W tiles,",
       "# UBLKCP = 1-D bulk copies (expert UP blocks), SYNCS = mbarrier operations, ATOMG/RED .64 = fixed-point accumulator updates.", ""]
for op, n in sorted(ops.items()):
    if op.startswith(SHOW):
        out.append(f"  {op:44s} {n}")
out.append(f"  {'total SASS instructions in the kernel':44s} {len(body)}")
idx = [i for i, l in enumerate(body) if "UTCHMMA" in l]
out += ["", "# --- the MMA issue loop (round 2: the whole warp issues, descriptors in uniform registers -- UIADD3 + UTCHMMA, no R2UR,",
        "#     no election loop; the TMA / bulk-copy producers further down still issue from one lane and show the ELECT ... BRA.U.ANY loop)"]
out += [l[:130] for l in body[max(0, idx[0] - 6): idx[-1] + 8]]
for op in ("LDTM", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "ATOMG.E.ADD.64", "RED.E.ADD.64"):
    hits = [i for i, l in enumerate(body) if op in l]
    if hits:
        out += ["", f"# --- first {op} and its neighbourhood"] + [l[:130] for l in body[max(0, hits[0] - 4): hits[0] + 4]]
whole = collections.Counter()
for k, b in funcs.items():
    for l in b:
        for op in ("UTCHMMA", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP"):
            if op in l:
                whole[op] += 1
out += ["", "# --- whole library: " + ", ".join(f"{op} {n}" for op, n in sorted(whole.items())),
        "# kernels: " + ", ".join(sorted({re.sub(r'^_ZN2af', '', k)[:40] for k in funcs if 'umma' in k}))[:900]]
open(os.path.join(ROOT, "profiles", f"{tag}_sass_switch_umma.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
