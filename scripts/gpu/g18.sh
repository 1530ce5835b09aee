python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_suite.py tests/test_gpu_train_aux.py -m gpu -x -q > gpurun_out/pytest_gpu18.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu18.log
timeout 1500 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3_18.json 2> gpurun_out/c3_18.err; echo "c3 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/c3_18.json')); print('c3', d['value'], d['e2e']['value'], d.get('extra',{}).get('e2e_graph'))"
