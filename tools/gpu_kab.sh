# cluster-size A/B for the latency configs: gpurun -- "bash tools/gpu_kab.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for C in 1 2 3; do
  for K in 2 4 8 16; do
    L1RXG_CLUSTER=$K timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/b$C.k$K.json 2> gpurun_out/$T/b$C.k$K.err
  done
  timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-companion --no-e2e > gpurun_out/$T/b$C.auto.json 2> gpurun_out/$T/b$C.auto.err
done
