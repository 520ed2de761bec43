"""Count SASS opcodes per function (and per innermost loop body) of a cubin/binary/.so."""
import re
import subprocess
import sys
from collections import Counter


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, funcs = None, {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
    return funcs


def opcode(ins):
    ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
    return ins.split()[0]


def loop_bodies(ins):
    """Backward branches: (target, branch) address ranges."""
    res = []
    for addr, text in ins:
        m = re.search(r"BRA\S*\s+(?:`?\(?\.L_x_\d+\)?|0x([0-9a-f]+))", text)
        m2 = re.search(r"0x([0-9a-f]+)", text) if "BRA" in text else None
        if m2:
            tgt = int(m2.group(1), 16)
            if tgt < addr:
                res.append((tgt, addr))
    return res


if __name__ == "__main__":
    path = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else ""
    for name, ins in functions(path).items():
        if pat not in name:
            continue
        c = Counter(opcode(t) for _, t in ins)
        print(f"== {name}: {len(ins)} instructions")
        print("   ", ", ".join(f"{k}:{v}" for k, v in c.most_common(14)))
        for lo, hi in loop_bodies(ins):
            body = [t for a, t in ins if lo <= a <= hi]
            cb = Counter(opcode(t) for t in body)
            spill = sum(v for k, v in cb.items() if k.startswith(("STL", "LDL")))
            print(f"   loop [{lo:#x},{hi:#x}] {len(body)} ins (local ld/st {spill}):",
                  ", ".join(f"{k}:{v}" for k, v in cb.most_common(12)))
