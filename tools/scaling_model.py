"""Fill model of the long-pair column-strip wavefront across G GPUs.

Every row strip of h rows sweeps all m columns in order, one column per warp step, so its
traversal takes m * t_step; a device keeps R = W_res * h rows in flight (W_res resident
warps) to run at full rate.  By Little's law, device g+1 lags device g by R rows of the
pipeline, and the last device finishes (G - 1) * R rows after the first: with T1 the one-GPU
time, T_G = T1 / G * (1 + (G - 1) * R / n)  =>  efficiency 1 / (1 + (G - 1) * R / n).
The measured per-step time (0.64 us per 1024-row task step on a loaded B200) gives
t_step = T1 / (S * G1 * W / W_res) consistently with the same formula.  The model is checked
on one GPU against virtual column strips (same code path) in tests/test_gpu_long*.py; the
multi-GPU numbers themselves are predictions (no multi-GPU box in this environment).
"""
import json
import sys


def efficiency(n: float, G: int, rows_per_warp: int, warps: int = 148 * 12) -> float:
    return 1.0 / (1.0 + (G - 1) * warps * rows_per_warp / n)


def main():
    n = float(sys.argv[1]) if len(sys.argv) > 1 else 5e6
    out = {}
    for h, rel in ((1024, 1.0), (512, 0.89)):  # NR = 16 / 8; rel = measured one-GPU rate
        out[f"{h}-row strips"] = {f"G={G}": round(efficiency(n, G, h) * rel, 3)
                                  for G in (1, 2, 4, 8)}
    need = 0.176 * n / (7 * 148 * 12)
    out["rows per warp for 85 % at G=8"] = round(need, 1)
    for n2 in (5e6, 20e6, 50e6, 250e6):
        out[f"n={n2:.0e}, 1024-row, G=8"] = round(efficiency(n2, 8, 1024), 3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
