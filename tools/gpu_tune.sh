# probe-stage sweep: bucket size (2^CG_BUCKET_LOG2 .. 2^(+1) cells) x filter extra bits
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
for bl in 0 1; do for fe in 4 5 6 7; do
  echo -n "bucket_log2=$bl fextra=$fe: "
  CG_BUCKET_LOG2=$bl CG_FILTER_EXTRA=$fe timeout 300 python tools/diag_stages.py 26 4 2>&1 | grep '"rep": 3' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_dict'], d['us_probe'], d['us_total'])"
done; done
