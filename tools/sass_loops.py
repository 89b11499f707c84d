"""List the loops (backward branches) of a kernel's SASS with their opcode
mix: the filter loops' per-iteration instruction accounting.

    python tools/sass_loops.py OBJ SUBSTR [min_len] [--listing START_HEX]"""
import collections
import re
import sys

from sass_fn import functions


def parse(body):
    ins = []
    for ln in body:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return ins


def opcode(text):
    t = text.split()
    i = 1 if t[0].startswith("@") else 0
    return t[i].split(".")[0]


def main():
    obj, sub = sys.argv[1], sys.argv[2]
    min_len = int(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else 40
    listing = None
    if "--listing" in sys.argv:
        listing = int(sys.argv[sys.argv.index("--listing") + 1], 16)
    for name, body in functions(obj):
        if sub not in name:
            continue
        ins = parse(body)
        addr = {a: k for k, (a, _) in enumerate(ins)}
        for k, (a, t) in enumerate(ins):
            m = re.search(r"\bBRA\b.*?(0x[0-9a-f]+)\s*$", t)
            if not m:
                continue
            tgt = int(m.group(1), 16)
            if tgt >= a or tgt not in addr:
                continue
            body_ins = ins[addr[tgt]:k + 1]
            if len(body_ins) < min_len:
                continue
            mix = collections.Counter(opcode(x) for _, x in body_ins)
            preds = sum(1 for _, x in body_ins if x.startswith("LOP3.LUT P"))
            print(f"loop 0x{tgt:04x}-0x{a:04x}: {len(body_ins)} instructions, LOP3 with predicate output {preds}: "
                  + " ".join(f"{o}:{c}" for o, c in mix.most_common()))
            if listing == tgt:
                for aa, x in body_ins:
                    print(f"    /*{aa:04x}*/ {x}")


if __name__ == "__main__":
    main()
