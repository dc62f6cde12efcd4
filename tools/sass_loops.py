"""Opcode histograms of the loops of one kernel's SASS (cuobjdump -sass -fun NAME obj).

  python tools/sass_loops.py OBJ KERNEL_SUBSTRING
Prints every backward-branch loop (start, end, instruction count, opcode histogram), so the
instruction cost of the inner edge loop can be checked here before spending GPU time."""
import collections
import re
import subprocess
import sys


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    names = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funs = [m for m in re.findall(r"Function : (\S+)", names) if pat in m]
    for f in funs:
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", f, obj], capture_output=True, text=True).stdout
        ins = []
        for ln in sass.splitlines():
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        print(f"== {f}: {len(ins)} instructions, STL {sum('STL' in t for _, t in ins)}, LDL {sum('LDL' in t for _, t in ins)}")
        for idx, (a, t) in enumerate(ins):
            m = re.search(r"BRA (?:\S+, )?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a:
                tgt = int(m.group(1), 16)
                body = [tt for aa, tt in ins if tgt <= aa <= a]
                c = collections.Counter()
                for tt in body:
                    op = re.sub(r"^@!?U?P\w+\s+", "", tt).split()[0].split(".")[0]
                    c[op] += 1
                print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr  " + " ".join(f"{k}:{v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main()
