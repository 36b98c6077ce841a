"""Probe NVML GPM NVLink throughput metrics on this box (field counters
138/139 report NOT_SUPPORTED on the pool's B200s)."""
import ctypes, time, traceback
import pynvml as p
import torch

p.nvmlInit()
h = p.nvmlDeviceGetHandleByIndex(0)
try:
    sup = p.c_nvmlGpmSupport_t()
    sup.version = p.NVML_GPM_SUPPORT_VERSION
    print("gpm support", p.nvmlGpmQueryDeviceSupport(h, sup).isSupportedDevice)
except Exception:
    traceback.print_exc()
try:
    s1, s2 = p.nvmlGpmSampleAlloc(), p.nvmlGpmSampleAlloc()
    p.nvmlGpmSampleGet(h, s1)
    x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
    if torch.cuda.device_count() > 1:
        y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
        t0 = time.perf_counter()
        for _ in range(20):
            y.copy_(x)
        torch.cuda.synchronize()
        print("copied 20 GiB 0->1 in", time.perf_counter() - t0)
    else:
        time.sleep(0.2)
    p.nvmlGpmSampleGet(h, s2)
    mg = p.c_nvmlGpmMetricsGet_t()
    mg.version = p.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = 2
    mg.sample1 = s1
    mg.sample2 = s2
    mg.metrics[0].metricId = p.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
    mg.metrics[1].metricId = p.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
    p.nvmlGpmMetricsGet(mg)
    for i in range(2):
        print("metric", mg.metrics[i].metricId, "ret", mg.metrics[i].nvmlReturn, "value", mg.metrics[i].value)
except Exception:
    traceback.print_exc()
