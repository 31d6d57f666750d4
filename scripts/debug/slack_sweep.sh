for sl in 0.5,64 1.0,64 1.0,128; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-parity --no-shuffled --bin-slack $sl > gpurun_out/slack_$sl.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/slack_$sl.json'))
print('$sl', round(d['value']/1e9,2), 'G/s ms/step', round(d['ms_per_step'],3), 'phase3', round(d['extra']['phase3_kernel_ms_per_step'],3), 'rebuilds', [s[4] for s in d['extra']['bin_stats']])"
done
