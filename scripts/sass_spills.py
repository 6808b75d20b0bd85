"""Local-memory (spill) instructions per source line, from `nvdisasm -g -c` output: sass_spills.py FILE.sass KERNEL_SUBSTR"""
import re, sys
fn = None; cur = None; stats = {}
for ln in open(sys.argv[1]):
    m = re.match(r'\s*\.text\.(\S+):', ln)
    if m:
        fn = m.group(1); continue
    m = re.search(r'//## File "(?:.*/)?([\w.]+)", line (\d+)', ln)
    if m:
        cur = m.group(1) + ':' + m.group(2); continue
    if fn and sys.argv[2] in fn and re.search(r'\b(STL|LDL)\b', ln):
        s = stats.setdefault(cur, [0, 0]); s[0 if 'STL' in ln else 1] += 1
for k, v in sorted(stats.items(), key=lambda x: -sum(x[1])):
    print(f"{k:30s} STL {v[0]:3d} LDL {v[1]:3d}")
