ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"sampler|straggler" python -c "
import torch,sys; sys.path.insert(0,'.')
from paper_2202_13927_b200.population import generate_population
d=torch.device('cuda',0)
for n,s in ((1000000,2),(100000,1)):
    generate_population(s, n, device=d, on_exhausted='redraw_weight')
" > gpurun_out/samp_ncu.csv 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/samp_ncu.csv')) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    print(r[h.index('Kernel Name')][:20], r[h.index('Metric Value')], r[h.index('Metric Unit')])
PY
