for v in base attnpark attnepi attnboth base; do
  for args in "--d 128 --bits 3 --variant full" "--d 256 --bits 3 --variant full"; do
    echo "$v $args $(IQ_LIB_PATH=paper_2603_28430_b200/build/var_$v/libisoquant.so python tools/attn_bench.py $args --heads 64 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k:(v["us"], round(v["keys_per_s"]/1e9,2)) for k,v in d.items() if k!="workload"})')"
  done
done
