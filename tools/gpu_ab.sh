# A/B of an env knob on the C5 stage timings: VAR=name VALS="a b"
python -c "from paper_1503_06029_b200 import build_lib; build_lib.build()"
for v in $VALS; do echo "== $VAR=$v"; env $VAR=$v timeout 300 python tools/diag_stages.py 26 5 2>&1 | grep '"rep": 4' | cut -c1-260; done
