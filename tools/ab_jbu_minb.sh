# A/B of VSBP_JBU_MINB builds (exp/libvsbp_minbM.so built with -DVSBP_JBU_MINB=M); run under gpurun
mkdir -p gpurun_out
for r in 1 2; do for m in 5 4 6; do
  if [ $m = 5 ]; then L=; else L=$PWD/exp/libvsbp_minb$m.so; fi
  VSBP_LIB=$L timeout 300 python tools/time_jbu.py --batch 128 --tag minb$m >> gpurun_out/ab_jbu.log 2>&1
done; done
for m in 5 4 6; do
  if [ $m = 5 ]; then L=; else L=$PWD/exp/libvsbp_minb$m.so; fi
  VSBP_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab_bench_$m.json 2>gpurun_out/ab_bench_$m.err
done
