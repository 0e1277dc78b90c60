mkdir -p gpurun_out
./tools/tmem_rate > gpurun_out/tmem_rate.txt 2>&1
for v in abl_ld abl_math; do
  MXM_LIB=$(pwd)/tools/variants/lib_$v.so timeout 300 python bench.py --config q2 --table w4a4_g128_sym --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --no-comparators > /tmp/b.json 2>/tmp/b.err
  echo "$v $(python -c 'import json; d=json.load(open("/tmp/b.json")); print(d["roofline"]["kernel_ms"])')" >> gpurun_out/tmem_rate.txt
done
cat gpurun_out/tmem_rate.txt
