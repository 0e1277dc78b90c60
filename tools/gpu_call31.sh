mkdir -p gpurun_out
timeout 1200 python tools/ablations.py gpurun_out/ablations.json > gpurun_out/ablations.log 2>&1; echo "abl rc=$?"
tail -5 gpurun_out/ablations.log
# compute-sanitizer on a small mixed layer (one call each tool)
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from synth import configs as C
from tests.moe_cases import make_case, gpu_layer, gpu_run
cfg = C.LayerConfig("san", 4, 1, 256, 512, 256, 2, 40)
t = [[C.WA(4, 128)] * 3, [C.WO(4, 128), C.WO(2, -1), C.WA(8, -1)], [C.WA(8, -1)] * 3, [C.WA(5, -1)] * 3, [C.WA(4, -1)] * 3]
case = make_case(cfg, t, 40, seed=1)
L = gpu_layer(case); y = gpu_run(L, case); print("ok", float(np.abs(y).max()))
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san.py > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.txt
  tail -3 gpurun_out/sanitizer_$tool.txt
done
