#!/bin/bash
# What NVLink counters does this box expose? (diagnostic)
nvidia-smi nvlink -s -i 0 2>&1 | head -20
nvidia-smi nvlink -gt d -i 0 2>&1 | head -40
nvidia-smi nvlink -gt r -i 0 2>&1 | head -10
python - <<'PY'
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
for name in ["NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX"]:
    fid = getattr(nv, name)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, scope, v.nvmlReturn, v.valueType, v.value.ullVal)
        except Exception as e:
            print(name, scope, "exc", e)
for name in dir(nv):
    if name.startswith("NVML_FI_DEV_NVLINK") and ("COUNT" in name or "BYTES" in name or "PKT" in name):
        print(name, getattr(nv, name))
PY
