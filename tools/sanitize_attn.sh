# compute-sanitizer over the attention kernel tests (both pool maps, NaN-filled pools) and smoke()
OUT=${OUT:-gpurun_out/sanattn}; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python -m pytest -x -q -p no:cacheprovider tests/test_kernels_gpu.py -k "paged_attention and (spec0 or spec1)" \
    > $OUT/attn_$tool.log 2>&1
  echo "attention tests $tool rc=$?" >> $OUT/summary.txt
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_memcheck.log 2>&1
echo "smoke memcheck rc=$?" >> $OUT/summary.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log >> $OUT/summary.txt
cat $OUT/summary.txt
