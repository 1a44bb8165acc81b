# pair stream-K hang hunt: debug build (bounded ring waits that report), 1024^3 and neighbours
set -x
export GEMM_F64_LIB=$PWD/paper_1706_10086_b200/libgemm_f64_dbg.so
timeout -s KILL 120 python tools/dbg_pair.py tma_64x64x32_w32x16_s6_pairsk 512,768,1024 > gpurun_out/r02_g37_dbg.txt 2>&1
echo rc=$?
timeout -s KILL 120 python tools/dbg_pair.py tma_64x64x32_w32x16_s4_pairsk,tma_64x64x16_w32x16_s8_pairsk 1024 >> gpurun_out/r02_g37_dbg.txt 2>&1
echo rc=$?
tail -40 gpurun_out/r02_g37_dbg.txt
unset GEMM_F64_LIB
timeout -s KILL 300 python tools/cfg_time.py plan,tma_64x64x32_w32x16_s6_pairsk,tma_64x64x32_w32x16_s4_pairsk,tma_64x64x16_w32x16_s8_pairsk 256,512,768,1024,2048,4096 > gpurun_out/r02_g37_pair.jsonl 2> gpurun_out/r02_g37_pair.err
cat gpurun_out/r02_g37_pair.jsonl
