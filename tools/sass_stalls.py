"""Per-region stall breakdown from an ncu source page (--print-source sass)."""
import csv, gzip, io, sys
f = sys.argv[1]
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows = list(csv.reader(io.TextIOWrapper(gzip.open(f), 'utf-8')))
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
keys = ['stall_no_inst', 'stall_long_sb', 'stall_wait', 'stall_barrier', 'stall_selected', 'stall_short_sb', 'stall_math', 'stall_mio', 'stall_lg']
def num(x):
    try: return float(x)
    except: return 0.0
n = len(data)
tot = {k: sum(num(r[col[k]]) for r in data) for k in keys}
print('total samples', {k: int(v) for k, v in tot.items()})
step = max(1, n // nb)
for b in range(0, n, step):
    seg = data[b:b+step]
    s = {k: int(sum(num(r[col[k]]) for r in seg)) for k in keys}
    ops = {}
    for r in seg:
        op = r[col['Source']].split()[0] if r[col['Source']].split() else ''
        if op.startswith('@'): op = r[col['Source']].split()[1]
        op = op.split('.')[0]
        ops[op] = ops.get(op, 0) + 1
    top = sorted(ops.items(), key=lambda x: -x[1])[:4]
    print(f'{b:6d}-{b+step:6d}', ' '.join(f'{k[6:]}={v}' for k, v in s.items() if v), '|', top)
