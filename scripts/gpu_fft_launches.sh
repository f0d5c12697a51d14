# F3 per-kernel times at C3 (ncu launch list of one hk_fft_matvec after a warm-up)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python scripts/fft_profile.py ${1:-C3} 1 > gpurun_out/fft_launch.csv 2>gpurun_out/fft_ncu.err
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/fft_launch.csv')) if len(r)>5]
hdr=None; data=[]
for r in rows:
    if r[0]=='ID': hdr=r; continue
    if hdr: data.append(r)
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
from collections import defaultdict
d=defaultdict(dict); names={}
for r in data:
    d[r[ii]][r[mi]]=r[vi]; names[r[ii]]=r[ki]
ks=[k for k in sorted(d, key=int) if any(s in names[k] for s in ('f1_','f2_','f3_'))]
for k in ks[len(ks)//2:]:
    m=d[k]
    print(names[k].split('(')[0].split('::')[-1][:28], 'us %.0f' % (float(m['gpu__time_duration.sum'])/1e3), 'rd %.2f GB' % (float(m['dram__bytes_read.sum'])/1e9), 'wr %.2f GB' % (float(m['dram__bytes_write.sum'])/1e9), 'fp64', m['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'], 'issue', m['smsp__issue_active.avg.pct_of_peak_sustained_active'], 'warps', m['sm__warps_active.avg.pct_of_peak_sustained_active'])
PY
