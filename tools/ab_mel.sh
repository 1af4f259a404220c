# A/B of the Mel workload on one box: tools/libnnab_ab.so (baseline build) vs the in-tree library
for i in 1 2 3; do
  for lib in tools/libnnab_ab.so paper_1912_12055_b200/libnnab.so; do
    NNAB_LIB=$lib timeout 200 python bench.py --workload mel --steps 100 --warmup 5 --no-breakdown 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])"
  done
done
