python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
tail -15 gpurun_out/gputest.log
python tools/time_ops.py --reps 30
python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['ops']), json.dumps(d['roofline']), d['gpu_launches'], d['clocks'])"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
