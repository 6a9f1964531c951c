for c in C1 C2 C3 C4 C5; do python bench.py --config $c --q 5 > gpurun_out/bench_all_$c.log 2>&1 || echo "bench $c failed"; tail -1 gpurun_out/bench_all_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
p=d['phases']
print(d['config']['workload'], 'step %.3f ms'%d['ms_per_step'], 'value %.2f'%d['value'], 'sketch %.2f [%s] (dominant frac %.3f)'%(d['sketch_tflops'], d['sketch_engine'], d['roofline']['frac']), 'qrcp %.3f solve %.3f gen %.2f est(q5) %.2f ms'%(p['qrcp_s']*1e3, p['solve_s']*1e3, p['generate_s']*1e3, p['error_estimate_s']*1e3), 'e2e %.2f'%d['e2e']['value'], 'tie %.3g'%d['tie_margin_min'], 'launches', d['gpu_launches'])
"; done
