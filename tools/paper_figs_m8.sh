# Fig. 11 analogue in the many-micro-batch regime (verdict r1 item 9): the same
# episode as tools/paper_figs.sh with 4 and 8 micro-batches, where a batch's
# prefetch has several steps of rotation to land in.
set -x
mkdir -p gpurun_out/figs
for m in 4 8; do
  W="--model qwen3-8b --requests 256 --prompt 512 --gen 128 --micro-batches $m --pool-frac 0.5 --resident-frac 0.5"
  timeout 1200 python -m paper_2605_02189_b200.cli compare $W --host-tokens 120000 \
      --policies dynamic,no_prefetch,static:0.5 --out gpurun_out/figs/compare_qwen3_8b_m$m.csv > gpurun_out/figs/compare_m$m.log 2>&1
  tail -5 gpurun_out/figs/compare_m$m.log
done
