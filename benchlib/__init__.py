"""bench.py's implementation (not product code): workloads, timing, clocks,
the whole-list oracle check and the reference arm.  The product package
``paper_2505_21194_b200`` never imports this package; this package may load
``oracle/`` (bench.py's parity check, cpu_baseline and --impl reference legs)."""
