timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for C in 0 16; do
  if [ $C = 0 ]; then unset P2G_WAVE_COLOURS; else export P2G_WAVE_COLOURS=$C; fi
  echo "== c3 wave $C"
  timeout 900 python bench.py --config c3 --no-cpu --no-e2e --steps 1 --warmup 1 | python -c "
import json,sys; d=json.load(sys.stdin); c=d['config']; r=d['roofline']
print('solves/s %.2f  ms/step %.1f  it mean %.1f max %d  iter_ms %.3f' % (d['value'], d['ms_per_step'], c['iterations_mean'], c['iterations_max'], r['iteration_ms']))
print({k: round(v['ms']*1e3,1) for k,v in r['classes'].items()})"
done
