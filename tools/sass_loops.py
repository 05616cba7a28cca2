"""Instruction mix of the hot loops of one kernel in an object file (SASS):
every backward branch whose body holds at least --min-fp64 DMUL/DADD/DFMA.

  python tools/sass_loops.py build/pgmres/planes.cu.o plane_ring_kernelILi1ELi27ELi2ELi1E
"""
import collections
import re
import subprocess
import sys


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    min_fp = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    on, ins = False, []
    for line in txt.splitlines():
        if "Function :" in line:
            on = pat in line
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if on and m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print(f"{pat}: {len(ins)} instructions")
    addr = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.\w+)*\s+(?:\w+,\s*)?0x([0-9a-f]+)", t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr:
            continue
        body = ins[addr[tgt]:i + 1]
        mix = collections.Counter()
        for _, b in body:
            op = b.split()[1] if b.startswith("@") else b.split()[0]
            mix[op.split(".")[0]] += 1
        fp = mix["DMUL"] + mix["DADD"] + mix["DFMA"]
        if fp < min_fp or len(body) > 600:  # innermost hot loops only
            continue
        print(f"loop {tgt:#x}..{a:#x}: {len(body)} instructions, fp64 {fp}: "
              + ", ".join(f"{k} {v}" for k, v in mix.most_common()))


if __name__ == "__main__":
    main()
