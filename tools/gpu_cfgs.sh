# bench lines of configs 1, 3, 5: gpurun -- "bash tools/gpu_cfgs.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for C in 1 3 5; do
  timeout 900 python bench.py --config $C > gpurun_out/$T/bench_config$C.json 2> gpurun_out/$T/bench_config$C.err
done
