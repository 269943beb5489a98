"""Mapped distributed executors for the paper's workloads (one process per GPU)."""
