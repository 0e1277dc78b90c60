#!/bin/bash
# quick perf pass: every config's block / GEMM time and roofline fraction (+ comparators for CMP configs)
mkdir -p gpurun_out; OUT=gpurun_out/perf${TAG}.txt; : > $OUT
for c in ${CFGS:-q2 q15 dsv2 mx}; do
  CMPF="--no-comparators"; case " ${CMP} " in *" $c "*) CMPF="";; esac
  timeout 400 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e $CMPF > gpurun_out/perf_$c$TAG.json 2>/tmp/b.err
  echo "$c rc=$? $(python -c '
import json,sys; d=json.load(open(sys.argv[1])); p=d["per_expert_roofline"]; c=d.get("comparators") or {}
cm=" ".join("%s=%.3f/%.3f" % (k[:22], v.get("block_ms",0), v.get("gemm_ms",0)) for k,v in c.items() if isinstance(v,dict))
print("step_ms=%.4f gemm_ms=%.4f frac=%.3f pe_frac=%.3f %s clk=%s" % (d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"], p["frac_of_gemm"], cm, d["clocks"].get("sm_mhz")))' gpurun_out/perf_$c$TAG.json 2>&1 | tail -1)" >> $OUT
done
for T in ${SMALLT}; do
  timeout 300 python bench.py --config mx --tokens $T --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-comparators > /tmp/b.json 2>/tmp/b.err
  echo "mx T=$T $(python -c 'import json; d=json.load(open("/tmp/b.json")); p=d["per_expert_roofline"]; print("step_ms=%.4f gemm_ms=%.4f t_roof_us=%.1f frac_gemm=%.3f" % (d["ms_per_step"], d["roofline"]["kernel_ms"], p["t_roof_us"], p["frac_of_gemm"]))' 2>&1 | tail -1)" >> $OUT
done
cat $OUT
