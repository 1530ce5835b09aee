"""Run ./peaks while sampling the SM clock with NVML; writes one JSON line (the measured
FP32 / FFMA2 / SFU peaks that bench.py's raster rooflines divide by)."""
import json
import os
import subprocess
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    import pynvml as nv

    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    clocks, stop = [], [False]

    def sample():
        while not stop[0]:
            clocks.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            time.sleep(0.01)

    t = threading.Thread(target=sample, daemon=True)
    t.start()
    out = subprocess.run([os.path.join(HERE, "peaks")], capture_output=True, text=True, check=True).stdout
    stop[0] = True
    t.join()
    res = json.loads(out.strip().splitlines()[-1])
    busy = [c for c in clocks if c > 0.5 * max(clocks)]
    res["sm_mhz_median"] = sorted(busy)[len(busy) // 2]
    res["sm_max_mhz"] = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
    res["gpu"] = nv.nvmlDeviceGetName(h)
    res["nominal_fp32_tflops_at_max"] = 148 * 128 * 2 * res["sm_max_mhz"] * 1e6 / 1e12
    print(json.dumps(res))


if __name__ == "__main__":
    main()
