# sweep prefix-index bucket size and filter resolution for the global probe (C5)
for bl in ${BLS:-0 1}; do for e in ${ES:-4 5 6}; do
  r=$(CG_FILTER_EXTRA=$e CG_BUCKET_LOG2=$bl python tools/diag_stages.py 26 3 2>&1 | sed -n 3p | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['us_dict'], d['us_probe'], d['us_total'])")
  echo "bucket_log2=$bl E=$e dict/probe/total_us: $r"
done; done
