# per-wave transition A/B (wave_trace.py, solve 2 of products eps=1e-7 and papers100M eps=1e-6)
o=gpurun_out/wave_ab.txt; : > $o
for shape in "products 1e-7" "papers100M 1e-6"; do
for env in "X=0" "GDIFF_WAVE_SERIAL=1" "GDIFF_WAVE_SERIAL=1 GDIFF_EXTRACT_BAL=1" "GDIFF_WAVE_SERIAL=1 GDIFF_RESET_MODE=1" "GDIFF_WAVE_SERIAL=1 GDIFF_RESET_MODE=2" "GDIFF_WAVE_SERIAL=1 GDIFF_RESET_MODE=3" "GDIFF_EXTRACT_BAL=1" "GDIFF_EXTRACT_BAL=1 GDIFF_RESET_MODE=3"; do
  echo "=== $shape $env" >> $o
  env $env timeout 600 python scripts/wave_trace.py $shape 2>&1 | sed -n '/solve 2/,$p' | python -c "
import sys,re
L=sys.stdin.read().splitlines()
k=[];e=[];r=[];n=[]
for l in L:
    m=re.match(r'wave (\d+) kernel ([\d.]+) us, extract done \+([\d.]+), reset done \+([\d.]+), next wave \+([\d.]+)',l)
    if m: k.append(float(m[2]));e.append(float(m[3]));r.append(float(m[4]));n.append(float(m[5]))
    if l.startswith('kernel ms'): print(l)
import statistics as s
print('waves',len(k),'kernel med %.1f  extract med %.1f  reset med %.1f  next med %.1f  sum next %.1f'%(s.median(k),s.median(e),s.median(r),s.median(n[:-1]),sum(n)))
" >> $o
done; done
echo "=== parity under the new forms" >> $o
GDIFF_EXTRACT_BAL=1 GDIFF_RESET_MODE=3 timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_xparity.py -x -q -m gpu 2>&1 | tail -3 >> $o
