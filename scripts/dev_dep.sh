# dev: deposit variants on the GEM bench (launch list per variant)
for d in ${DEPS:-0 1 2 3 4}; do
  BP_F32_DEPOSIT=$d timeout 300 ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/dep_var$d.csv python bench.py --steps 10 --warmup 0 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
done
