"""Find scoreboard sharing between shared-memory loads and global loads in a kernel's SASS:
an instruction that waits on scoreboard k for the result of a load (shared or global) although a
global load issued after it also holds k -- the wait then lasts that later load's round trip
(the v6 finding: column reads behind the chunk's first gathers, K1). Prints each such place.

    cuobjdump -sass libmcinv.so > k.sass; python tools/sass_sbcheck.py k.sass [kernel-substring]
"""
import re
import sys


def parse(lines):
    i, out = 0, []
    while i < len(lines) - 1:
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* 0x([0-9a-f]{16}) \*/', lines[i])
        if m:
            m2 = re.match(r'\s*/\* 0x([0-9a-f]{16}) \*/', lines[i + 1])
            c = int(m2.group(1), 16) >> 41
            out.append((int(m.group(1), 16), m.group(2).strip(), (c >> 5) & 7, (c >> 11) & 0x3f))
            i += 2
            continue
        i += 1
    return out


def false_waits(blk):
    """(address, instruction, scoreboard, kind) of every wait in one function's SASS that
    needs an earlier load's result while a later global load holds the same scoreboard."""
    ins = parse(blk.splitlines())
    out = []
    last = {}

    def regs(txt):
        return set(int(r) for r in re.findall(r"\bR(\d+)\b", txt))

    for addr, op, wb, wm in ins:
        body = re.sub(r"^@!?U?P\d+\s+", "", op)
        mnem = body.split()[0]
        operands = body[len(mnem):]
        for k in range(6):
            if wm >> k & 1:
                pend = last.get(k, [])
                src = regs(operands.split(",", 1)[1] if "," in operands else operands)
                need = [n for n, p in enumerate(pend) if p[1] & src]
                if need and [p for p in pend[need[-1] + 1:] if p[0] == "LDG"]:
                    out.append((addr, op, k, pend[need[-1]][0]))
                last[k] = []
        if wb != 7:
            kind = "LDG" if mnem.startswith("LDG") else ("LDS" if mnem.startswith("LDS") else "other")
            dst = operands.split("desc")[0] if kind == "LDG" else operands.split(",")[0]
            last.setdefault(wb, []).append((kind, regs(dst)))
    return out


def main():
    text = open(sys.argv[1]).read().split("Function : ")
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    for blk in text[1:]:
        name = blk.split("\n", 1)[0].strip()
        if want not in name:
            continue
        ins = parse(blk.splitlines())
        last = {}  # sb -> [(kind, dest registers)] written since the last wait on it
        hits = 0

        def regs(txt):
            return set(int(r) for r in re.findall(r"\bR(\d+)\b", txt))

        for addr, op, wb, wm in ins:
            body = re.sub(r"^@!?U?P\d+\s+", "", op)
            mnem = body.split()[0]
            operands = body[len(mnem):]
            for k in range(6):
                if wm >> k & 1:
                    pend = last.get(k, [])
                    src = regs(operands.split(",", 1)[1] if "," in operands else operands)
                    need = [n for n, p in enumerate(pend) if p[1] & src]
                    if need:
                        # a false dependency: the value comes from an earlier load, but a global
                        # load issued after it on the same scoreboard must return first
                        later = [p for p in pend[need[-1] + 1:] if p[0] == "LDG"]
                        if later:
                            hits += 1
                            if hits <= 8:
                                print(f"  {addr:05x} {op[:60]} waits sb{k}: {pend[need[-1]][0]} value behind a later global load")
                    last[k] = []
            if wb != 7:
                kind = "LDG" if mnem.startswith("LDG") else ("LDS" if mnem.startswith("LDS") else "other")
                dst = operands.split("desc")[0] if kind == "LDG" else operands.split(",")[0]
                last.setdefault(wb, []).append((kind, regs(dst)))
        print(f"{name[:90]}: {hits} shared/global scoreboard waits")


if __name__ == "__main__":
    main()
