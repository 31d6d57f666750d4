cp paper_2008_04397_b200/libbp_b200.so /tmp/lib_default.so
for v in s3 s4 s6; do
  cp build_variants/lib_$v.so paper_2008_04397_b200/libbp_b200.so
  for B in 1048576 2097152; do
    BP_HOST_BATCH=$B timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu --no-parity --no-shuffled > gpurun_out/hs.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/hs.json')); print('$v', $B, round(d['e2e']['value']/1e9,3))"
  done
done
cp /tmp/lib_default.so paper_2008_04397_b200/libbp_b200.so
