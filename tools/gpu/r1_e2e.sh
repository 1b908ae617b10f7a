mkdir -p gpurun_out
for cfg in "3 64" "4 64" "2 128" "3 128" "4 128" "3 32" "4 256"; do
  set -- $cfg; KB_STAGE_SLOTS=$1 KB_STAGE_MB=$2 timeout 300 python tools/e2e_probe.py | sed "s/^/slots=$1 mb=$2 /"
done
