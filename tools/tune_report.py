import json, re, sys
for line in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/tune.log'):
    if line.startswith('==='): print(line.strip()); continue
    if line.startswith('[prof]'):
        m = re.search(r'ms=\s*([\d.]+)', line)
        if m and float(m.group(1)) > 1.0: print('   ', line.strip())
        continue
    if line.startswith('{'):
        d = json.loads(line)
        print('   ms/step=%.2f iters=%s frac=%.3f launches=%d' % (d['ms_per_step'], d['config']['iters_per_solve'], d['roofline']['frac'], d['gpu_launches']))
    elif line.strip(): print('   !!', line.strip()[:200])
