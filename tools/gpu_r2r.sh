# round 2: parity fields of the config 1/2/3/5 lines
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for C in 2 3 1 5; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/$T/bench_config$C.json 2> gpurun_out/$T/bench_config$C.err
done
