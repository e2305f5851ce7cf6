# per-kernel durations of one pipeline run (ncu, serialised): bash tools/gpu/ktimes.sh C3 [env...]
cfg=$1; shift
env "$@" ncu --metrics gpu__time_duration.sum,launch__block_size,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:'sweep4|prior_select' python tools/prof_once.py $cfg 2>/dev/null | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
d=collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ix['ID']],r[ix['Kernel Name']][:60]),{})[r[ix['Metric Name']]]=r[ix['Metric Value']]
for k,v in d.items(): print(k[1], v)
"
