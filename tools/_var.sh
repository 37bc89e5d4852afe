# kernel-variant A/B: bench config 1 with each build, interleaved
for rep in 1 2; do
for v in default a b c; do
  if [ $v = default ]; then unset RS_LIB_PATH; else export RS_LIB_PATH=$PWD/paper_2505_12663_b200/_lib/var/$v.so; fi
  timeout 300 python bench.py --steps 30 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1e3,2), round(d['value']/1e6,1), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
done; done
