# config-3 cluster sweep: gpurun -- "bash tools/gpu_k3.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for K in 4 6 8; do
  L1RXG_CLUSTER=$K timeout 300 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/$T/b3_k$K.json 2> gpurun_out/$T/b3_k$K.err
done
for K in 8 12 16; do
  L1RXG_CLUSTER=$K timeout 300 python bench.py --config 1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/$T/b1_k$K.json 2> gpurun_out/$T/b1_k$K.err
done
