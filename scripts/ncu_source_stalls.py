"""Per-SASS-line stall attribution from an ncu source-page CSV (debug aid, not product).
   ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv ; python scripts/ncu_source_stalls.py src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[ix['# Samples']]) for r in data)
print('total samples', tot)
agg = {s: sum(f(r[ix[s]]) for r in data) for s in stalls}
for s, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f'{s:28s} {v:8.0f} {100 * v / tot:5.1f}%')
print()
for r in sorted(data, key=lambda r: -f(r[ix['# Samples']]))[:ntop]:
    st = sorted(((f(r[ix[s]]), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{f(r[ix['# Samples']]):6.0f} {f(r[ix['Instructions Executed']]):9.0f} wf={r[ix['L1 Wavefronts Shared']]:>8s} "
          f"{r[ix['Source']][:60]:60s} " + ' '.join(f'{n}={v:.0f}' for v, n in st))
print('instr executed', sum(f(r[ix['Instructions Executed']]) for r in data))
print('smem wavefronts', sum(f(r[ix['L1 Wavefronts Shared']]) for r in data), 'ideal',
      sum(f(r[ix['L1 Wavefronts Shared Ideal']]) for r in data))
