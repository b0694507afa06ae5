mkdir -p gpurun_out
V2=$(realpath paper_1603_08081_b200/_lib/libfourierbf_b200_v2.so)
FBF_LIBRARY=$V2 timeout 300 python tools/sanitize_cases.py > gpurun_out/v2_cases.log 2>&1; echo "cases rc=$?" >> gpurun_out/v2_cases.log
FBF_LIBRARY=$V2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_device.py -x -q > gpurun_out/v2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v2_pytest.log
CONFIGS="c2 c5 c1 c3" ROUNDS=2 bash tools/ab.sh paper_1603_08081_b200/_lib/libfourierbf_b200.so paper_1603_08081_b200/_lib/libfourierbf_b200_v2.so > gpurun_out/v2_ab.txt 2>&1
cat gpurun_out/v2_cases.log; tail -3 gpurun_out/v2_pytest.log; cat gpurun_out/v2_ab.txt
