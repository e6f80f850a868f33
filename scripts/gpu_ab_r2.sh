# Round-2 kernel A/B: parity of the test variant, then alternating bench runs.
# env: TESTV (variant to test), VARIANTS (bench list; "name" or "name:poly"
# for an exp-poly split override), RUNS (default 2), BENCH_ARGS
mkdir -p gpurun_out
rm -f gpurun_out/quick.log
# a hung or wrong variant must cost seconds, not the call: quick check first
OKV=""
for spec in ${VARIANTS} ${TESTV}; do
  v="${spec%%:*}"
  case " $OKV " in *" $v "*) continue;; esac
  if BSA_LIB_VARIANT=$v timeout -s KILL 90 python scripts/quick_check.py >> gpurun_out/quick.log 2>&1; then
    OKV="$OKV $v"
  else
    echo "variant $v FAILED quick check" >> gpurun_out/quick.log
  fi
done
case " $OKV " in *" $TESTV "*) ;; *) TESTV="";; esac
if [ -n "$TESTV" ]; then
  BSA_LIB_VARIANT=$TESTV timeout -s KILL 400 python -m pytest tests/test_gpu_attention.py \
    tests/test_gpu_shard.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance.py tests/test_gpu_key_ranges.py -x -q 2>&1 | tail -5 > gpurun_out/t_ab_$TESTV.log
fi
rm -f gpurun_out/ab2_*.txt
for r in $(seq 1 ${RUNS:-2}); do
for spec in ${VARIANTS}; do
  v="${spec%%:*}"; poly=""; [ "$spec" != "$v" ] && poly="${spec#*:}"
  case " $OKV " in *" $v "*) ;; *) continue;; esac
  tag=$(echo "$spec" | tr ':' '_')
  if [ -n "$poly" ]; then export BSA_TC_EXP_POLY=$poly; else unset BSA_TC_EXP_POLY; fi
  BSA_LIB_VARIANT=$v timeout -s KILL 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-dense $BENCH_ARGS 2>/dev/null | tail -1 >> gpurun_out/ab2_$tag.txt
done; done
unset BSA_TC_EXP_POLY
python scripts/ab2_report.py $(for s in ${VARIANTS}; do echo "$s" | tr ':' '_'; done) > gpurun_out/ab_report.txt
