# multi-GPU bench lines (torchrun), N from $1, workloads in the rest
N=$1; shift
for w in "$@"; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --workload $w --no-cpu-baseline > gpurun_out/r2_bench_${w}_${N}gpu.json 2> gpurun_out/r2_bench_${w}_${N}gpu.err
  tail -1 gpurun_out/r2_bench_${w}_${N}gpu.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', $N, round(d['ms_per_step'],3), d['rank_evaluate_ms'], d['e2e']['stage1_solve_s'])" || tail -5 gpurun_out/r2_bench_${w}_${N}gpu.err
done
