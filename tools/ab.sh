L=paper_2204_02348_b200/lib
for r in 1 2 3; do for v in old new; do cp $L/libholo_b200.so.$v $L/libholo_b200.so; for c in ${CONFIGS:-dualpol}; do python bench.py --config $c --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', '$c', round(d['value']/1e6,3))"; done; done; done
cp $L/libholo_b200.so.new $L/libholo_b200.so
