"""Opcode histogram of the innermost loops of one kernel's SASS (cuobjdump -sass output).

    python tools/sass_loops.py kernel.sass [min_len]

A loop is a backward branch; its body is [target, branch]. Prints each loop of at least
min_len instructions with its opcode counts (the hot loop of a generation kernel is the
unrolled step pair)."""
import collections
import re
import sys


def parse(path):
    ins = []
    for line in open(path):
        m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)([^;]*);', line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    return ins


def main():
    ins = parse(sys.argv[1])
    min_len = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    addr_idx = {a: i for i, (a, _, _) in enumerate(ins)}
    for i, (a, op, args) in enumerate(ins):
        if not op.startswith("BRA"):
            continue
        m = re.search(r'0x([0-9a-f]+)', args)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr_idx:
            continue
        body = ins[addr_idx[tgt]:i + 1]
        if len(body) < min_len:
            continue
        c = collections.Counter(o.split('.')[0] for _, o, _ in body)
        print(f"loop {tgt:#x}..{a:#x}: {len(body)} instructions")
        print("  " + ", ".join(f"{k} {v}" for k, v in sorted(c.items(), key=lambda x: -x[1])))


if __name__ == "__main__":
    main()
