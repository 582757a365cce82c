# Scratch driver for gpurun sweeps (edited per experiment): gpurun --timeout 1500 -- "bash tools/gpu_sweep.sh"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step'])" $1 "$2"; }
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for bw in 0 1; do
L1RXG_BWARP=$bw python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b2.log 2>&1; summ gpurun_out/b2.log "config2 bwarp=$bw"
L1RXG_BWARP=$bw python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b3.log 2>&1; summ gpurun_out/b3.log "config3 bwarp=$bw"
L1RXG_BWARP=$bw python bench.py --config 1 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b1.log 2>&1; summ gpurun_out/b1.log "config1 bwarp=$bw"
done
