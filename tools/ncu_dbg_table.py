"""Table of per-launch k_conv3x3_tc durations from tools/_ncu_dbg.sh CSVs."""
import csv
import io
import sys

modes = [int(m) for m in sys.argv[1:]] or [0, 31]
labels = ['fwdL2', 'fwdL3', 'fwdL4', 'fwdL5', 'fwdL6', 'fwdL7', 'fwdL8', 'dgL8', 'dgL7', 'dgL6',
          'dgL5', 'dgL4', 'dgL3', 'dgL2', 'valL2', 'valL3']
rows = {}
for d in modes:
    txt = open(f'gpurun_out/ncu_dbg{d}.csv').read()
    r = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
    rows[d] = [(x['Kernel Name'].split('<')[1].split('>')[0], float(x['Metric Value']))
               for x in r if x['Metric Name'] == 'gpu__time_duration.sum']
print('kernel          ' + ' '.join(f'{d:>7}' for d in rows))
for j, (n, _) in enumerate(rows[modes[0]]):
    print(f'{labels[j]:6} {n:9}' + ' '.join(f'{rows[d][j][1] / 1000:7.1f}' for d in rows))
