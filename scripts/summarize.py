"""Summarise a gpu_round.sh tag: bench line, launch list, ncu full metrics."""
import csv, json, subprocess, sys
tag = sys.argv[1]
d = json.loads(open(f"gpurun_out/{tag}_bench.log").read().strip().splitlines()[-1])
print(f"value {d['value']/1e9:.1f} Gsteps/s  step {d['ms_per_step']:.3f} ms  kernel {d['roofline']['kernel_ms']:.3f} ms  "
      f"frac {d['roofline']['frac']:.3f}  e2e {d['e2e']['value']/1e9:.1f} Gsteps/s ({d['e2e']['ms_per_step']:.2f} ms)  "
      f"clocks {d['clocks']}  launches {d['gpu_launches']}")
if 'cpu_baseline' in d: print('cpu', d['cpu_baseline'])
try:
    rows = [r for r in csv.reader(l for l in open(f"gpurun_out/{tag}_launches.csv") if not l.startswith('=='))]
    h = rows[0]
    ks = [dict(zip(h, r)) for r in rows[1:]]
    ks = [k for k in ks if k.get('Metric Name') == 'gpu__time_duration.sum']
    print('launches:', ' '.join(f"{k['Kernel Name'][6:18]}:{float(k['Metric Value'])/1e3:.1f}" for k in ks if 'rasp' in k['Kernel Name'])[:600])
except FileNotFoundError:
    pass
try:
    raw = subprocess.run(['ncu', '-i', f'gpurun_out/{tag}_prof.ncu-rep', '--page', 'raw', '--csv'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    want = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
            'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
            'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__registers_per_thread',
            'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
            'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']
    for r in rows[2:]:
        print(' '.join(f"{w.split('__')[1][:22]}={r[h.index(w)]}" for w in want if w in h))
except Exception as e:
    print('no ncu', e)
