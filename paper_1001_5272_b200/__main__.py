"""python -m paper_1001_5272_b200 <tft|itft|multiply|bench|selftest> ... (the `tftmul` CLI)."""
from .cli import entry

entry()
