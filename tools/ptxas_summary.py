"""Per-kernel registers / stack / spills from a ptxas -v report (csrc/ptxas_info.txt)."""
import re
import subprocess
import sys


def parse(text):
    out, cur = {}, None
    for ln in text.splitlines():
        m = re.search(r"Compiling entry function '(\w+)'", ln) or re.search(r"Function properties for (\w+)", ln)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m and cur:
            out.setdefault(cur, {}).update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", ln)
        if m and cur:
            out.setdefault(cur, {})["regs"] = int(m.group(1))
    return out


def demangle(n):
    try:
        return subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    except Exception:
        return n


if __name__ == "__main__":
    txt = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2310_17274_b200/csrc/ptxas_info.txt").read()
    for k, v in sorted(parse(txt).items()):
        if "regs" in v:
            name = demangle(k)
            name = re.sub(r"\(.*\)", "", name.replace("(anonymous namespace)::", ""))
            print(f"{name:60s} regs={v['regs']:3d} stack={v.get('stack', 0):4d} spill={v.get('spill_st', 0)}/{v.get('spill_ld', 0)}")
