mkdir -p gpurun_out
python tools/pcie_probe.py > gpurun_out/pcie_probe.txt 2>&1; cat gpurun_out/pcie_probe.txt
for mi in 0 16 64 256; do
  echo "piece_mi=$mi"; IZG_HOST_PIECE_MI=$mi python tools/e2e_probe.py 16384 2>&1 | tail -2
done
