mkdir -p gpurun_out
CMD="python tools/run_pipeline.py --config ${CFG:-C3} --reps 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/prof_plain.log
python3 - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches.csv')) if len(r)>5]
hdr=rows[0]; iN=hdr.index('Kernel Name'); iM=hdr.index('Metric Name'); iV=hdr.index('Metric Value'); iI=hdr.index('ID')
from collections import OrderedDict
k=OrderedDict()
for r in rows[1:]:
    k.setdefault(r[iI], [r[iN][:38]]).append(f"{r[iM].split('.')[0][-22:]}={r[iV]}")
for i,v in k.items(): print(i, ' | '.join(v))
PY
