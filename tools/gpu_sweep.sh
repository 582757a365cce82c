# Scratch driver for gpurun sweeps (edited per experiment): gpurun --timeout 1500 -- "bash tools/gpu_sweep.sh"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step'])" $1 "$2"; }
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1
python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-companion > gpurun_out/b2.log 2>&1; summ gpurun_out/b2.log "config2"
python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b3.log 2>&1; summ gpurun_out/b3.log "config3"
python bench.py --config 4 --recordings 256 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw4.log 2>&1; summ gpurun_out/sw4.log "config4-256"
