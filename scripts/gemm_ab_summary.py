"""Summarise scripts/gpu_gemm_ab.sh captures (ncu --clock-control base): per
GEMM kind, ours / cuBLAS in kilo-cycles (duration x SM clock, so boxes with
different base clocks compare) and tensor-pipe active %.

    python scripts/gemm_ab_summary.py gpurun_out/ab
"""
import csv,glob,collections,sys,statistics
for f in sorted(glob.glob(sys.argv[1]+'/*.csv')):
    rows=[r for r in csv.reader(l for l in open(f) if l.startswith('"'))]
    if not rows: print(f,'empty'); continue
    h=rows[0]; d=rows[1:]
    ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iid=h.index('ID')
    per=collections.defaultdict(dict)
    for r in d: per[int(r[iid])][r[im]]=float(r[iv].replace(',',''))
    ids=sorted(per)
    out=collections.defaultdict(list)
    for j,i in enumerate(ids):
        kind=['fwd1','fwd2','dgelu','wgrad'][(j//2)%4]; who='ours' if j%2==0 else 'cub'
        m=per[i]; out[(kind,who)].append((m['gpu__time_duration.sum']*m['sm__cycles_elapsed.avg.per_second']/1e9/1e3, m['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']))
    s=f.split('/')[-1][:-4].ljust(14)
    for kind in ['fwd1','fwd2','dgelu','wgrad']:
        o=out[(kind,'ours')]; c=out[(kind,'cub')]
        s+=f" {kind}: {statistics.median(x[0] for x in o):5.0f}/{statistics.median(x[0] for x in c):5.0f}kc {statistics.median(x[1] for x in o):4.1f}/{statistics.median(x[1] for x in c):4.1f}%"
    print(s)
