import glob, json, re, collections
res = collections.defaultdict(list)
for f in sorted(glob.glob('gpurun_out/abn*.json')):
    v = re.match(r'gpurun_out/abn(.*)\.\d+\.json', f).group(1) or 'default'
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        res[v].append((round(d['ms_per_step'], 4), round(d['latency_ms_per_frame'], 4), round(d['stages_ms_eager']['unet'], 4)))
    except Exception as e:
        res[v].append(('err', str(e)[:60]))
for v, r in res.items():
    print(f"{v:12s}", r)
