"""Remove a retired compile-time experiment switch from a source file, keeping
the code of its default value (a minimal unifdef for `#if NAME`, `#if !NAME`,
`#if NAME == v` / `#elif NAME == v` / `#else` / `#endif` chains whose conditions
name only that macro; any other #if is left alone and tracked for nesting).

  python tools/strip_switch.py FILE NAME VALUE
"""
import re
import sys


def strip(lines, name, value):
    out = []
    # stack entries: None for a foreign #if (kept verbatim), else a dict for ours
    stack = []

    def active():
        return all(e is None or e["keep"] for e in stack)

    def evaluate(cond):
        cond = cond.strip()
        m = re.fullmatch(rf"!\s*{name}", cond)
        if m:
            return value == 0
        m = re.fullmatch(rf"{name}", cond)
        if m:
            return value != 0
        m = re.fullmatch(rf"{name}\s*==\s*(\d+)", cond)
        if m:
            return value == int(m.group(1))
        return None

    for ln in lines:
        s = ln.strip()
        m = re.match(r"#\s*if\s+(.*)$", s)
        if m and not s.startswith("#ifdef") and not s.startswith("#ifndef"):
            v = evaluate(m.group(1))
            if v is None:
                stack.append(None)
                if active():
                    out.append(ln)
            else:
                stack.append({"keep": v, "taken": v})
            continue
        if s.startswith("#ifdef") or s.startswith("#ifndef"):
            stack.append(None)
            if active():
                out.append(ln)
            continue
        m = re.match(r"#\s*elif\s+(.*)$", s)
        if m and stack and stack[-1] is not None:
            v = evaluate(m.group(1))
            if v is None:
                raise SystemExit(f"mixed #elif condition: {s}")
            e = stack[-1]
            e["keep"] = (not e["taken"]) and v
            e["taken"] = e["taken"] or v
            continue
        if s.startswith("#else") and stack and stack[-1] is not None:
            e = stack[-1]
            e["keep"] = not e["taken"]
            e["taken"] = True
            continue
        if s.startswith("#endif") and stack:
            e = stack.pop()
            if e is None and active():
                out.append(ln)
            continue
        if active():
            out.append(ln)
    return out


if __name__ == "__main__":
    path, name, value = sys.argv[1], sys.argv[2], int(sys.argv[3])
    with open(path) as f:
        lines = f.readlines()
    res = strip(lines, name, value)
    # drop the switch's own #ifndef/#define/#endif default block
    txt = "".join(res)
    txt = re.sub(rf"#ifndef {name}\n#define {name} [^\n]*\n#endif\n", "", txt)
    with open(path, "w") as f:
        f.write(txt)
