#!/bin/bash
# CUDA-core GEMV probe vs the tcgen05 path at tiny m (w4a16-g128, Mixtral expert shapes)
mkdir -p gpurun_out; O=gpurun_out/gemv; mkdir -p $O
timeout 120 ./tools/variants/gemv_probe 14336 4096 > $O/probe.txt 2>&1
for T in 1 4 8; do
  timeout 300 python bench.py --config mx --table w4a16_g128_asym --tokens $T --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-comparators > /tmp/g.json 2>/dev/null
  python -c "
import json; d=json.load(open('/tmp/g.json')); p=d['per_expert_roofline']; g=d['roofline']['kernel_ms']
print('mx w4a16-g128 T=$T: gemm %.1f us, alg bytes %.1f MB -> %.2f TB/s, per-expert frac %.3f' % (g*1e3, p['alg_bytes']/1e6, p['alg_bytes']/(g*1e-3)/1e12, p['frac_of_gemm']))" >> $O/probe.txt
done
cat $O/probe.txt
