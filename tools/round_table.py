"""Per-round kernel times (ns) of the last complete solve in an ncu launch
list (host loop): python tools/round_table.py launches.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
seq = []
for r in rows:
    if 'Kernel Name' in r:
        h = r
        continue
    if h and len(r) == len(h) and r[h.index('Metric Name')] == 'gpu__time_duration.sum':
        seq.append((r[h.index('Kernel Name')], float(r[h.index('Metric Value')].replace(',', ''))))
idx = [i for i, (k, v) in enumerate(seq) if 'k_reset' in k]
s = seq[idx[-2]:idx[-1]]
short = {'k_sell<1, 1': 'dense', 'k_sell<1, 0': 'wl', 'k_split_finish': 'split', 'k_cand': 'cand',
         'k_commit_list': 'clist', 'k_commit': 'commit', 'k_mark<': 'mark', 'k_mark(': 'mark'}
rnd, cur = [], {}
for k, v in s:
    name = k.split('(')[0].replace('void ', '').replace('pgb::', '')
    if name.startswith('k_sell<1, 1') or name.startswith('k_sell<0, 1'):
        if cur:
            rnd.append(cur)
        cur = {}
    for p, t in short.items():
        if (name + '(').startswith(p) or name.startswith(p):
            cur[t] = cur.get(t, 0) + v
            break
rnd.append(cur)
tot = 0
for i, c in enumerate(rnd):
    t = sum(c.values())
    tot += t
    print(f"{i + 1:3d} " + ' '.join(f"{k}={v / 1e3:7.1f}" for k, v in c.items()) + f"  sum={t / 1e3:7.1f} us")
print(f"total {tot / 1e3:.1f} us")
