"""Opcode mix of a kernel's hottest loop, from cuobjdump -sass of an object.

  python tools/sass_mix.py paper_2603_28430_b200/build/kinst_full_f16.cu.o \
      '_ZN2iq8k_encodeI6__halfLi128ELi3ELi0ELi1ELb0E'

Finds the function whose mangled name starts with the given prefix, locates
the backward branches (loops), and prints the opcode histogram of the
largest loop body (the per-row-pair loop of the stage-1 kernels).  Static
analysis only: no GPU needed.
"""
import collections
import re
import subprocess
import sys


def sass_of(obj, prefix):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if name.startswith(prefix):
            return name, f
    raise SystemExit(f"no function {prefix}")


INS = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)([^;]*);")


def parse(body):
    ins = []
    for m in INS.finditer(body):
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    return ins


def loops(ins):
    out = []
    for addr, op, args in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", args)
            if t and int(t.group(1), 16) < addr:
                out.append((int(t.group(1), 16), addr))
    return out


def main():
    obj, prefix = sys.argv[1], sys.argv[2]
    name, body = sass_of(obj, prefix)
    ins = parse(body)
    ls = loops(ins)
    print(name, "instructions:", len(ins), "loops:", [(hex(a), hex(b), sum(1 for x in ins if a <= x[0] <= b)) for a, b in ls])
    if not ls:
        return
    a, b = max(ls, key=lambda ab: sum(1 for x in ins if ab[0] <= x[0] <= ab[1]))
    if len(sys.argv) > 3:
        a, b = ls[int(sys.argv[3])]
    body = [x for x in ins if a <= x[0] <= b]
    h = collections.Counter(op.split(".")[0] + ("2" if ".F32x2" in op or "2" in op.split(".")[0][-1:] else "") for _, op, _ in body)
    full = collections.Counter(op for _, op, _ in body)
    print(f"loop {hex(a)}..{hex(b)}: {len(body)} instructions")
    for k, v in full.most_common():
        print(f"  {v:5d}  {k}")


if __name__ == "__main__":
    main()
