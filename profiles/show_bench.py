"""Print the key fields of a bench.py JSON line (usage: python profiles/show_bench.py FILE)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"value {d['value']/1e6:.3f} M tok/s  ms/step {d['ms_per_step']:.3f}  "
      f"gemm {d['roofline']['achieved']:.0f} TF/s frac {d['roofline']['frac']:.3f}  "
      f"exposed {d.get('exposed_a2a_ms')}  clocks {d.get('clocks')}")
if 'e2e' in d:
    print(f"e2e {d['e2e']['value']/1e6:.3f} M tok/s")
for k, v in d.get('kernels', {}).items():
    extra = f"{v['tflops']:7.0f} TF/s" if 'tflops' in v else (f"{v['gbs']:7.0f} GB/s ({v['hbm_frac']:.2f})" if 'gbs' in v else "")
    us = v.get('us', v.get('span_us', 0.0))
    print(f"  {k:20s} {us:8.1f} us  " + (extra or ("(side-stream span)" if 'span_us' in v else "")))
print(f"  sum of in-line ops {sum(v.get('us', 0.0) for v in d.get('kernels', {}).values()):.1f} us")
