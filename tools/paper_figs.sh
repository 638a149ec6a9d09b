# Hardware analogues of the paper's policy comparison (Fig. 11: tokens/s of
# dynamic vs no_prefetch vs static prefetch through the episode loop) and
# per-iteration residency series (Fig. 12, `cli report`), Qwen3-8B shape on
# one B200.  Outputs under gpurun_out/figs/ (copied to profiles/figs/).
set -x
mkdir -p gpurun_out/figs
W="--model qwen3-8b --requests 256 --prompt 512 --gen 128 --micro-batches 2 --pool-frac 0.5 --resident-frac 0.5"
timeout 900 python -m paper_2605_02189_b200.cli compare $W --host-tokens 120000 \
    --policies dynamic,no_prefetch,static:0.5 --out gpurun_out/figs/compare_qwen3_8b.csv > gpurun_out/figs/compare.log 2>&1
timeout 600 python -m paper_2605_02189_b200.cli decode $W --trace gpurun_out/figs/decode_trace.jsonl \
    --metrics gpurun_out/figs/decode_metrics.json > gpurun_out/figs/decode.log 2>&1
timeout 120 python -m paper_2605_02189_b200.cli report --trace gpurun_out/figs/decode_trace.jsonl \
    --out gpurun_out/figs/report_qwen3_8b.csv >> gpurun_out/figs/decode.log 2>&1
rm -f gpurun_out/figs/decode_trace.jsonl
cat gpurun_out/figs/compare.log gpurun_out/figs/decode.log | tail -20
