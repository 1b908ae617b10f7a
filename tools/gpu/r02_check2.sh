mkdir -p gpurun_out
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 30 build/sanitize/kb_sanitize quick > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; grep -E "SUMMARY|kb_sanitize:" gpurun_out/sanitize_$t.log
  grep -oE "in void kb::[a-z0-9_]+<[^(]*" gpurun_out/sanitize_$t.log | sort | uniq -c | sort -rn | head -20
done
python tools/e2e_probe.py 4194304 pinned
python tools/e2e_probe.py 4194304 pageable
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2000 gpurun_out/bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
for k in ('value','ms_per_step','roofline','e2e','e2e_pageable','gpu_launches','clocks'): print(k, d.get(k))
for e in d['extra']: print(e)
PY
