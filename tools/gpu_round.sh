#!/usr/bin/env bash
# One GPU call: GPU tests, the bench line, the ncu launch list of a short bench
# run and one `--set full` capture per hot-path kernel. Everything lands in
# gpurun_out/ (copy the summaries worth keeping into profiles/).
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag] [parts]'
#   parts: comma list of probe,smoke,tests,bench,launches,k1,k2,k4,k8 (default all)
set -u
TAG=${1:-r1}
PARTS=${2:-probe,smoke,tests,bench,launches,k1,k2,k4,k8}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
has() { [[ ",$PARTS," == *",$1,"* ]]; }
nproc > "$OUT/nproc.txt"
nvidia-smi -q -d CLOCK > "$OUT/clocks_start.txt" 2>&1
if has probe; then timeout 300 python tools/probe_box.py > "$OUT/probe.log" 2>&1; cp gpurun_out/probe_box.json "$OUT/" 2>/dev/null; fi
if has smoke; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"; fi
if has tests; then timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"; fi
if has bench; then timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"; fi
NCU="ncu --clock-control none"
if has tptests; then timeout 900 python -m pytest tests/test_gpu_tp_loopback.py tests/test_gpu_tp_ipc.py tests/test_gpu_ckpt.py tests/test_gpu_hostpool.py tests/test_gpu_fusion.py -q > "$OUT/pytest_tp_ckpt.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_tp_ckpt.log"; fi
if has decode; then
  timeout 300 python tools/decode_probe.py 39 4237 12 > "$OUT/decode_probe.json" 2> "$OUT/decode_probe.err"
  timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/decode_launches.csv" \
    python tools/decode_probe.py 39 4237 3 > "$OUT/decode_ncu.log" 2>&1
fi
if has k1ab; then
  timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > "$OUT/pytest_attention.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_attention.log"
  for shape in "39 4237" "8 4237" "64 4224" "128 2000" "200 1000" "16 16000"; do
    for mode in 0 1; do
      CS_K1_SPLITK=$mode timeout 300 python tools/decode_probe.py $shape 8 >> "$OUT/k1ab.jsonl" 2>> "$OUT/k1ab.err"
      echo "{\"mode_splitk\": $mode, \"shape\": \"$shape\"}" >> "$OUT/k1ab.jsonl"
    done
  done
  timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/decode_launches_sk.csv" \
    python tools/decode_probe.py 39 4237 3 > "$OUT/decode_ncu_sk.log" 2>&1
fi
if has gemmab; then
  timeout 900 python -m pytest tests/test_gpu_wgemm.py -x -q > "$OUT/pytest_wgemm.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_wgemm.log"
  CS_K7_SK=1 timeout 600 python tools/gemm_k7.py 50 > "$OUT/gemm_sk.jsonl" 2> "$OUT/gemm_sk.err"
  CS_K7_SK=0 timeout 600 python tools/gemm_k7.py 50 > "$OUT/gemm_cluster.jsonl" 2> "$OUT/gemm_cluster.err"
  for w in 2 1 0; do
    CS_WGEMM=$w timeout 300 python tools/decode_probe.py 39 4237 8 >> "$OUT/decode_wgemm.jsonl" 2>> "$OUT/decode_wgemm.err"
    echo "{\"wgemm\": $w}" >> "$OUT/decode_wgemm.jsonl"
  done
  CS_WGEMM=1 timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/decode_launches_k7.csv" \
    python tools/decode_probe.py 39 4237 3 > "$OUT/decode_ncu_k7.log" 2>&1
fi
if has k2ab; then
  timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > "$OUT/pytest_attention.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_attention.log"
  timeout 600 python tools/k2_sweep.py 20 > "$OUT/k2_1cta.jsonl" 2> "$OUT/k2_1cta.err"
  CS_K2_PAIR=1 timeout 600 python tools/k2_sweep.py 20 > "$OUT/k2_pair.jsonl" 2> "$OUT/k2_pair.err"
  CS_K2_PAIR=1 timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > "$OUT/pytest_attention_pair.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_attention_pair.log"
fi
if has k1st; then
  timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > "$OUT/pytest_attention.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_attention.log"
  CS_K1_STAGES=3 timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -k k1 > "$OUT/pytest_attention3.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_attention3.log"
  for shape in "39 4237" "8 4237" "16 16000" "24 4000"; do
    for st in 2 3; do
      CS_K1_STAGES=$st timeout 300 python tools/decode_probe.py $shape 8 >> "$OUT/k1st.jsonl" 2>> "$OUT/k1st.err"
      echo "{\"stages\": $st, \"shape\": \"$shape\"}" >> "$OUT/k1st.jsonl"
    done
  done
fi
if has hosttimers; then
  CS_HOST_TIMERS=1 timeout 900 python bench.py --no-probes --legs "" > "$OUT/bench_ht.json" 2> "$OUT/bench_ht.err"
fi
if has stream; then
  timeout 300 ./tools/stream_bench > "$OUT/stream_bench.jsonl" 2>&1
fi
if has k1wv; then
  for shape in "39 4237" "24 4000" "50 4300"; do
    for wv in 1 2 4; do
      CS_K1_SK_WAVES=$wv timeout 300 python tools/decode_probe.py $shape 8 >> "$OUT/k1wv.jsonl" 2>> "$OUT/k1wv.err"
      echo "{\"waves\": $wv, \"shape\": \"$shape\"}" >> "$OUT/k1wv.jsonl"
    done
  done
  CS_K1_SK_WAVES=2 timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -k k1 > "$OUT/pytest_k1wv.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_k1wv.log"
fi
if has fusionab; then
  timeout 900 python tools/fusion_ab.py 5 > "$OUT/fusion_ab.jsonl" 2> "$OUT/fusion_ab.err"
  CS_NO_FUSE=0 timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/fusion_launches_on.csv" \
    python tools/fusion_ab.py child 8192 1 > /dev/null 2>&1
  CS_NO_FUSE=1 timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file "$OUT/fusion_launches_off.csv" \
    python tools/fusion_ab.py child 8192 1 > /dev/null 2>&1
fi
if has dump; then
  timeout 900 python bench.py --no-probes --legs "" --dump "$OUT/iters.npz" > "$OUT/bench_dump.json" 2> "$OUT/bench_dump.err"
fi
if has attn; then
  timeout 900 python -m pytest tests/test_gpu_attention.py -q > "$OUT/pytest_attention.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_attention.log"
fi
if has models; then
  timeout 1500 python bench.py --workload qwen14b --no-probes --no-cpu --legs "" > "$OUT/bench_qwen14b.json" 2> "$OUT/bench_qwen14b.err"
  timeout 2400 python bench.py --workload llama70b --no-probes --no-cpu --legs "" > "$OUT/bench_llama70b.json" 2> "$OUT/bench_llama70b.err"
fi
if has k1rope; then
  for shape in "39 4237" "8 4237" "64 2000"; do
    for nf in 1 0; do
      CS_NO_FUSE=$nf timeout 300 python tools/decode_probe.py $shape 10 >> "$OUT/k1rope.jsonl" 2>> "$OUT/k1rope.err"
      echo "{\"no_fuse\": $nf, \"shape\": \"$shape\"}" >> "$OUT/k1rope.jsonl"
    done
  done
fi
if has fusiontest; then
  timeout 900 python -m pytest tests/test_gpu_fusion.py -q > "$OUT/pytest_fusion.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_fusion.log"
fi
if has wgemmab; then
  for shape in "39 4237" "16 4237" "56 4300"; do
    for w in 2 1 0; do
      CS_WGEMM=$w timeout 300 python tools/decode_probe.py $shape 10 >> "$OUT/wgemmab.jsonl" 2>> "$OUT/wgemmab.err"
      echo "{\"wgemm\": $w, \"shape\": \"$shape\"}" >> "$OUT/wgemmab.jsonl"
    done
  done
fi
if has k7pdl; then
  for shape in "39 4237" "56 4300"; do
    for np in 0 1; do
      CS_K7_NO_PDL=$np timeout 300 python tools/decode_probe.py $shape 10 >> "$OUT/k7pdl.jsonl" 2>> "$OUT/k7pdl.err"
      echo "{\"no_pdl\": $np, \"shape\": \"$shape\"}" >> "$OUT/k7pdl.jsonl"
    done
    CS_WGEMM=0 timeout 300 python tools/decode_probe.py $shape 10 >> "$OUT/k7pdl.jsonl" 2>> "$OUT/k7pdl.err"
    echo "{\"no_pdl\": \"cublas\", \"shape\": \"$shape\"}" >> "$OUT/k7pdl.jsonl"
  done
fi
if has waitab; then
  for wb in 0 1 0 1; do
    CS_WAIT_BLOCK=$wb timeout 900 python bench.py --no-probes --legs "" --no-cpu >> "$OUT/waitab.jsonl" 2>> "$OUT/waitab.err"
    echo "{\"wait_block\": $wb}" >> "$OUT/waitab.jsonl"
  done
fi
if has k1thr; then
  for shape in "56 4300" "64 4224" "80 3000" "100 2500" "128 2000"; do
    for thr in default 100000; do
      if [ "$thr" = default ]; then unset CS_K1_SK_PAIRS; else export CS_K1_SK_PAIRS=$thr; fi
      timeout 300 python tools/decode_probe.py $shape 10 >> "$OUT/k1thr.jsonl" 2>> "$OUT/k1thr.err"
      echo "{\"thr\": \"$thr\", \"shape\": \"$shape\"}" >> "$OUT/k1thr.jsonl"
    done
  done
  unset CS_K1_SK_PAIRS
fi
if has launches; then
  CS_NO_PACING=1 CS_PROFILE_REGION=1 timeout 1200 $NCU --profile-from-start off --metrics gpu__time_duration.sum -c 8000 --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 12 --warmup 3 --no-cpu --no-probes > "$OUT/launches_bench.log" 2>&1
fi
if has k1; then
  timeout 600 $NCU --set full --import-source on -k regex:attn_decode_kernel -s 1 -c 1 -o "$OUT/k1_decode" -f \
    python tools/ncu_targets.py decode > "$OUT/k1.log" 2>&1
fi
if has k1sk; then
  timeout 600 $NCU --set full --import-source on -k regex:attn_decode -s 1 -c 1 -o "$OUT/k1sk_decode" -f \
    python tools/ncu_targets.py decode 3 39 4237 > "$OUT/k1sk.log" 2>&1
fi
if has k2; then
  timeout 600 $NCU --set full --import-source on -k regex:attn_prefill -s 1 -c 1 -o "$OUT/k2_prefill" -f \
    python tools/ncu_targets.py prefill > "$OUT/k2.log" 2>&1
fi
if has k8; then
  timeout 600 $NCU --set full --import-source on -k regex:gemm_pf -s 4 -c 1 -o "$OUT/k8_gemm" -f \
    python tools/ncu_targets.py gemm > "$OUT/k8.log" 2>&1
fi
if has k4; then
  timeout 600 $NCU --set full --import-source on -k regex:"kv_pack|kv_move" -c 1 -o "$OUT/k4_gather" -f \
    python tools/ncu_targets.py gather > "$OUT/k4.log" 2>&1
fi
nvidia-smi -q -d CLOCK > "$OUT/clocks_end.txt" 2>&1
echo done
