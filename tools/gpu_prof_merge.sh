python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
mkdir -p gpurun_out
CHUNK_BITS=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_merge_buckets -c 1 -o gpurun_out/merge -f python tools/dist_stages.py 24 8 > /dev/null 2>&1
