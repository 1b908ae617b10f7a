# Host staging probes: memcpy bandwidth, PCIe ceilings, e2e pinned / pageable sweeps.
mkdir -p gpurun_out
g++ -O3 -march=native -pthread tools/microbench/memcpy_bw.cpp -o /tmp/memcpy_bw && /tmp/memcpy_bw
python tools/pcie_probe.py
for kind in pinned pageable; do
  for mb in 64 128 256; do
    for slots in 3 4; do
      echo "KB_STAGE_MB=$mb KB_STAGE_SLOTS=$slots"; KB_STAGE_MB=$mb KB_STAGE_SLOTS=$slots timeout 120 python tools/e2e_probe.py 4194304 $kind
    done
  done
done
for ct in 4 8 12 16; do echo "KB_COPY_THREADS=$ct"; KB_COPY_THREADS=$ct timeout 120 python tools/e2e_probe.py 4194304 pageable; done
