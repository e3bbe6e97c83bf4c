import sys, torch
sys.path.insert(0, ".")
import datagen, paper_1104_2732_b200 as cp
x = datagen.make("dup256", 1 << 28, "f32", device="cuda")
v, info = cp.median(x, return_info=True)
print(v, info)
for r in cp.get_trace():
    print(r["kind"], r["t"], r["c_lt"] if r["c_lt"] < 2**63 else "U", r["c_eq"] if r["c_eq"] < 2**63 else "U", r["interior"], r["scanned"], r["written"], r["compacted"])
