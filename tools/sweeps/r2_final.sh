# driver-style round-end run: GPU tests, smoke, default bench, reference arm
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "gpu suite rc=$?"; tail -2 gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_c3.err; echo "c3 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_c3.json').read().strip().splitlines()[-1]); print('C3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'], d['cpu_baseline'].get('reference_numba',{}).get('value'))"
