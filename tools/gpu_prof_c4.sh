# ncu --set full captures of the C4 (ell = 1024) kernels
set -x
mkdir -p gpurun_out
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
for k in ${KERNELS:-k_gather_dedupe k_probe_global k_onesweep}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/c4_$k -f python tools/configs_timing.py ${CFG:-C4} 1 > gpurun_out/ncu_c4_$k.log 2>&1
done
ls gpurun_out
