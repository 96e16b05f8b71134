"""mrsolve-b200 (placeholder; full API wired below)."""
