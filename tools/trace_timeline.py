"""Timeline of one DPP_TRACE step: start/end per scope, sorted by start, by host thread."""
import re, sys
lines = open(sys.argv[1]).read().split("\n")
step = sys.argv[2] if len(sys.argv) > 2 else "2"
on = False
ev = []
for l in lines:
    if l.startswith("---- step"):
        on = l.split()[-1] == step
        continue
    m = re.match(r"\[dpp-trace\] (\S+)\s+([\d.]+) ms .*@\s*([\d.]+) t(\d+)", l)
    if on and m:
        ev.append((float(m.group(3)) * 1e3 if float(m.group(3)) < 1e4 else float(m.group(3)), m.group(1), float(m.group(2)), m.group(4)))
if not ev:
    sys.exit("no events")
t0 = min(e[0] for e in ev)
for s, n, d, t in sorted(ev):
    if n.startswith("gmres.") and n != "gmres.total":
        continue
    print(f"{(s - t0):9.3f} {(s - t0 + d):9.3f}  {d:7.3f}  t{t}  {n}")
