# A/B of two prebuilt libraries (gpurun_out/libs/base.so vs $VARIANT.so): c2 pipelined + sequential, c3 sequential
L=paper_2305_18396_b200/lib/libhelinear.so
for rep in 1 2; do
for v in base ${VARIANT:-nz8}; do
  cp gpurun_out/libs/$v.so $L
  for mode in "" --sequential; do
    timeout 300 python bench.py --no-cpu-baseline --no-attention --steps 40 $mode > /tmp/c.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/c.json')); print('$v c2 $mode', d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
  done
  timeout 600 python bench.py --config c3 --plan --sequential --no-cpu-baseline --no-attention --steps 3 > /tmp/c.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/c.json')); print('$v c3', d['value'])"
done
done
cp gpurun_out/libs/base.so $L
