# ncu of the same lat_layer_kernel launches under two builds (ab/lib_old.so, ab/lib_new.so)
for v in old new; do
CORAL_S1_LIB=$PWD/ab/lib_$v.so ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:lat_layer_kernel -s 48 -c 4 --csv --log-file gpurun_out/ab_$v.csv python tools/profile_eval.py c2 --solves 2 > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/ab_$v.csv"))); hdr=None
for r in rows:
    if "Kernel Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print("$v", d["ID"], d["Metric Name"][:30], d["Metric Value"])
PY
done
