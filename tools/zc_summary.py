"""Summarise gpurun_out/zc_<variant>.csv (tools/fused_zc.sh): per fused template, total ms, DRAM GB,
mean L2 hit rate and DRAM % of peak; plus the first cycle's per-launch times."""
import csv
import glob
import io
import sys
from collections import defaultdict


def load(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    launches = defaultdict(dict)
    for r in rows:
        key = (int(r['ID']), r['Kernel Name'])
        v = r['Metric Value'].replace(',', '')
        launches[key][r['Metric Name']] = float(v)
    return [(k[1], m) for k, m in sorted(launches.items())]


for path in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/zc_*.csv')):
    L = load(path)
    print('==', path, len(L), 'launches')
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    for name, m in L:
        short = name[name.find('<'):name.find('>') + 1] if '<' in name else name
        a = agg[short]
        a[0] += 1
        a[1] += m.get('gpu__time_duration.sum', 0) / 1e6
        a[2] += m.get('dram__bytes_read.sum', 0) / 1e9
        a[3] += m.get('lts__t_sector_hit_rate.pct', 0)
        a[4] += m.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0)
    tot = 0
    for s, a in sorted(agg.items()):
        tot += a[1]
        print(f'  {s:24s} n={a[0]:4d} ms={a[1]:9.2f} GB={a[2]:9.1f} hit={a[3]/a[0]:5.1f}% dram={a[4]/a[0]:5.1f}%')
    print(f'  total ms {tot:.1f}')
    print('  first 31:', ' '.join(f"{m.get('gpu__time_duration.sum', 0)/1e6:.2f}" for _, m in L[:31]))
