# Round-2 (third session) evidence, part A: smoke, bench x2, reference arm,
# launch list, ncu --set full summaries of the headline fused kernel (b = 3, 4),
# the quantizer and fused + codes (reports kept in /tmp, summaries here).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_s3.log
for i in 1 2; do timeout 900 python bench.py > gpurun_out/bench_s3_$i.json 2> gpurun_out/bench_s3_$i.err; echo "bench $i rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_s3.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s3.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-e2e --no-kernels --no-traffic > gpurun_out/b_ncu_s3.log 2>&1; echo "launches rc=$?"
for spec in "roundtrip 3" "roundtrip 4" "quantize 3" "roundtrip_emit 3"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encode -c 1 -o /tmp/s3_$1_b$2 python tools/launch_kernels.py --kernel $1 --bits $2 --reps 2 > gpurun_out/ncu_s3_$1_b$2.log 2>&1; echo "ncu $1 b$2 rc=$?"
  python tools/ncu_summary.py /tmp/s3_$1_b$2.ncu-rep --stalls --json gpurun_out/ncu_s3_$1_b$2.json > /dev/null 2>&1
done
du -sh gpurun_out
