# A/B timing of builds of libcoral_s1.so on one box: bash tools/ab_bench.sh [variants...]
# (default: old new -> ab/lib_old.so, ab/lib_new.so), two rounds, bench.py --steps 10.
VARS="${*:-old new}"
for i in 1 2 3; do for v in $VARS; do
CORAL_S1_LIB=$PWD/ab/lib_$v.so python bench.py --no-cpu-baseline --no-c5 --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), round(d['stage_ms']['evaluate'],3), round(d['stage_ms']['enumerate'],3), round(d['roofline']['launch_ms'],4), round(d['roofline_top']['launch_ms'],4))"
done; done
