"""Which NVML NVLink byte counters does this box expose?  Copies 4 GiB GPU1 -> GPU0 (copy engines over
NVLink) and prints every candidate counter before / after, per link, so bench.py reads the right one.

    python tools/microbench/nvlink_probe.py      (2+ GPUs)
"""
import json

import pynvml
import torch


def fields(h):
    out = {}
    for name in ("NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES",
                 "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX",
                 "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX"):
        fid = getattr(pynvml, name, None)
        if fid is None:
            continue
        per = []
        for link in range(18):
            try:
                v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                per.append(int(v.value.ullVal) if v.nvmlReturn == 0 else f"ret{v.nvmlReturn}")
            except Exception as e:  # noqa: BLE001
                per.append(type(e).__name__)
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [fid])[0]
            agg = int(v.value.ullVal) if v.nvmlReturn == 0 else f"ret{v.nvmlReturn}"
        except Exception as e:  # noqa: BLE001
            agg = type(e).__name__
        out[name] = {"links": per, "noscope": agg}
    return out


def main():
    pynvml.nvmlInit()
    h0 = pynvml.nvmlDeviceGetHandleByIndex(0)
    before = fields(h0)
    a = torch.empty(1 << 29, dtype=torch.float64, device="cuda:1")  # 4 GiB
    b = torch.empty(1 << 29, dtype=torch.float64, device="cuda:0")
    a.fill_(1.0)
    torch.cuda.synchronize(1)
    b.copy_(a)
    torch.cuda.synchronize(0)
    after = fields(h0)
    print(json.dumps({"before": before, "after": after, "bytes_copied": a.numel() * 8}, indent=0))


if __name__ == "__main__":
    main()
