JB_PROFILE=1 timeout 900 python tools/exp_build_prof.py 500000 960 > gpurun_out/c3_prof.log 2>&1
python - <<'PY'
import re
tot={}
rows=[l for l in open('gpurun_out/c3_prof.log') if l.startswith('[jb] batch [')]
for l in rows:
    for k,v in re.findall(r'(\w+) ([\d.]+)ms',l): tot[k]=tot.get(k,0)+float(v)
print({k:round(v,1) for k,v in tot.items()})
PY
grep "^build" gpurun_out/c3_prof.log | cut -c1-70
ncu --set full --import-source on --clock-control none -k regex:"owner_(merge|matrix)_kernel" --launch-skip 12 -c 1 -o gpurun_out/prof_owner_c3m python tools/exp_build_prof.py 500000 960 > gpurun_out/ncu_owner_c3.log 2>&1
tail -2 gpurun_out/ncu_owner_c3.log
