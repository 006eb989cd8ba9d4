"""Partial preprocessor: resolve #if/#ifdef/#ifndef/#elif/#else/#endif blocks
whose conditions involve only the given macros (fixed to their production
values), drop those macros' '#ifndef X / #define X v / #endif' default blocks,
and substitute them in remaining code.  Used once to retire measured-and-
rejected build switches from the product sources (their A/B results are in
profiles/r01_experiments.md and r02_experiments.md).

    python tools/unifdef.py FILE... -D FL_X=1 -D FL_Y=0
"""
import re
import sys


def evaluate(expr, vals):
    e = expr
    e = re.sub(r"defined\s*\(\s*(\w+)\s*\)", lambda m: "1" if m.group(1) in vals else "0", e)
    toks = re.findall(r"[A-Za-z_]\w*", e)
    for t in toks:
        if t not in vals:
            return None
    for k, v in sorted(vals.items(), key=lambda kv: -len(kv[0])):
        e = re.sub(rf"\b{k}\b", str(v), e)
    e = e.replace("&&", " and ").replace("||", " or ").replace("!", " not ").replace("not =", "!=")
    try:
        return bool(eval(e))
    except Exception:
        return None


def process(lines, vals):
    out = []
    # stack entries: (mode, taken) mode: 'keep' = unresolved (emit directives), 'res' = resolved
    stack = []
    emitting = lambda: all(s["emit"] for s in stack)  # noqa: E731
    i = 0
    while i < len(lines):
        ln = lines[i]
        st = ln.strip()
        m = re.match(r"#\s*(ifndef|ifdef|if|elif|else|endif)\b(.*)", st)
        # default block: #ifndef X / #define X v / #endif for a resolved macro
        if m and m.group(1) == "ifndef" and m.group(2).strip().split("//")[0].strip() in vals:
            name = m.group(2).strip().split("//")[0].strip()
            j = i + 1
            while j < len(lines) and not lines[j].strip().startswith("#endif"):
                j += 1
            i = j + 1
            continue
        if not m:
            if emitting():
                for k, v in vals.items():
                    if re.search(rf"\b{k}\b", ln) and not st.startswith("#define " + k):
                        ln = re.sub(rf"\b{k}\b", str(v), ln)
                out.append(ln)
            i += 1
            continue
        d, rest = m.group(1), m.group(2).split("//")[0].strip()
        if d in ("if", "ifdef", "ifndef"):
            if d == "ifdef":
                r = True if rest in vals else None
            elif d == "ifndef":
                r = False if rest in vals else None
            else:
                r = evaluate(rest, vals)
            parent = emitting()
            if r is None:
                stack.append({"res": False, "emit": True, "done": False})
                if parent:
                    out.append(ln)
            else:
                stack.append({"res": True, "emit": r, "done": r})
        elif d == "elif":
            top = stack[-1]
            if top["res"]:
                r = evaluate(rest, vals)
                if r is None:
                    raise SystemExit(f"unresolvable #elif after a resolved #if: {st}")
                top["emit"] = (not top["done"]) and r
                top["done"] = top["done"] or r
            else:
                stack.pop()
                parent = emitting()
                stack.append(top)
                if parent:
                    out.append(ln)
        elif d == "else":
            top = stack[-1]
            if top["res"]:
                top["emit"] = not top["done"]
                top["done"] = True
            else:
                stack.pop()
                parent = emitting()
                stack.append(top)
                if parent:
                    out.append(ln)
        elif d == "endif":
            top = stack.pop()
            if not top["res"] and emitting():
                out.append(ln)
        i += 1
    return out


if __name__ == "__main__":
    files, vals = [], {}
    args = sys.argv[1:]
    k = 0
    while k < len(args):
        if args[k] == "-D":
            n, v = args[k + 1].split("=")
            vals[n] = int(v)
            k += 2
        else:
            files.append(args[k])
            k += 1
    for f in files:
        src = open(f).read().split("\n")
        open(f, "w").write("\n".join(process(src, vals)))
