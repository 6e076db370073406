set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not sanitizer and not two_ranks and not single_rank" > gpurun_out/pytest_r02b.log 2>&1; tail -5 gpurun_out/pytest_r02b.log
RAAS_LIB=build_exp/libraas_s20d1.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "lockstep or bitwise or sanitizer or roundtrip" > gpurun_out/pytest_r02b_s20d1.log 2>&1; tail -3 gpurun_out/pytest_r02b_s20d1.log
bash scripts/ab.sh "--steps 100;--config 4 --steps 60;--config 2 --steps 200;--steps 60 --score quest" 2 build_exp/libraas_base.so build_exp/libraas_s20d1.so build_exp/libraas_s16d1.so build_exp/libraas_s20d1b8.so 2>&1 | tee gpurun_out/ab_r02b.txt
