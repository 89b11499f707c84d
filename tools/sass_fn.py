"""Print the SASS of the function(s) whose mangled name contains SUBSTR.

    python tools/sass_fn.py OBJ SUBSTR [--mix]
--mix prints the opcode histogram instead of the listing."""
import collections
import re
import subprocess
import sys


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    cur, body = None, []
    for ln in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(ln)
    if cur:
        yield cur, body


def main():
    obj, sub = sys.argv[1], sys.argv[2]
    for name, body in functions(obj):
        if sub not in name:
            continue
        ins = [ln for ln in body if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln)]
        if "--mix" in sys.argv:
            c = collections.Counter(re.sub(r"^\s*/\*[0-9a-f]+\*/\s*(@!?U?P\w+\s+)?", "", ln).split()[0].split(".")[0]
                                    for ln in ins)
            print(name, len(ins), " ".join(f"{k}:{v}" for k, v in c.most_common(30)))
        else:
            print("\n".join(ins))


if __name__ == "__main__":
    main()
