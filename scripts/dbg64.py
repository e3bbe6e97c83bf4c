import sys, torch
sys.path.insert(0, ".")
import datagen, paper_1104_2732_b200 as cp
x = datagen.make("uniform", 1 << 28, "f64", device="cuda")
for cap in (0, 1 << 20):
    cp.set_config(select_cap=cap, record_trace=1)
    try:
        v, info = cp.median(x, return_info=True)
        print(cap, "ok", v, info["passes"], info["exit"], info["z_count"])
    except Exception as e:
        print(cap, "ERR", e)
    for r in cp.get_trace():
        print("   ", {k: r[k] for k in ("kind", "t", "c_lt", "c_eq", "interior", "scanned", "written")})
xs = x.sort().values
print("true", float(xs[(x.numel() + 1) // 2 - 1]))
