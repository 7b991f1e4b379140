#!/bin/bash
# Re-create the round-2 evidence under profiles/ on one B200 (run from the repo
# root inside gpurun; outputs land in gpurun_out/, copy the ones you want).
#   gpurun --timeout 5400 -- 'bash tools/reproduce_r02.sh'
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider                         > gpurun_out/gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()"                          > gpurun_out/smoke.log 2>&1
python bench.py                                                             > gpurun_out/r02_bench.json 2>&1
python bench.py --impl reference                                            > gpurun_out/r02_bench_reference.json 2>&1
python tools/config_sweep.py                                                > gpurun_out/r02_config_sweep.jsonl 2>&1
python tools/hmv_phases.py                                                  > gpurun_out/r02_hmv_phases.jsonl 2>&1
python tools/graph_small.py                                                 > gpurun_out/r02_graph_small.jsonl 2>&1
python tools/rank_parity.py                                                 > gpurun_out/r02_rank_parity.txt 2>&1
python tools/c5_readiness.py rung1                                          > gpurun_out/r02_c5_rung1.json 2>&1
python tools/c5_readiness.py part0                                          > gpurun_out/r02_c5_part0_of_8.json 2>&1
MVTAG=_r02 bash tools/mv16_launches.sh                                      > gpurun_out/r02_mv16_launches.txt 2>&1
bash tools/ncu_mv16_sweeps.sh
bash tools/sanitize.sh
ncu --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum \
    --kernel-name-base function -k "regex:^k_(orth|project|sumsq|weights|trunc|jacobi|svd|compact)" --csv \
    --log-file gpurun_out/exec_flops_c3.csv python tools/compress_exec_flops.py run 3 1048576 4 1e-6
python tools/compress_exec_flops.py sum gpurun_out/exec_flops_c3.csv        > gpurun_out/r02_compress_exec_flops_c3.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-compress                      > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02_launches.csv                  > gpurun_out/r02_launches_summary.txt
python tools/compress_timeline.py 3 1048576 4 1e-6 2 seq                    > gpurun_out/r02_compress_timeline_c3.txt 2>&1
bash tools/ncu_bsr_mv_tma.sh                                                # -> gpurun_out/bsr_tma.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:k_bsr_tma -s 1 -c 1 -o gpurun_out/r02_k_bsr_tma \
    python tools/microbench/c4_hmv.py 3                                     > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/tma_stream tools/microbench/tma_stream.cu -lcuda \
    && ./tools/microbench/tma_stream                                        > gpurun_out/r02_tma_stream.txt 2>&1
python tools/microbench/compressed_hmv.py                                   > gpurun_out/r02_compressed_hmv.json 2>&1
python tools/microbench/compressed_mv16.py                                  > gpurun_out/r02_compressed_mv16.json 2>&1
