"""Seeded synthetic inputs (host mirror in host.py, device twin in datagen.cu).
Shared test/bench infrastructure; holds none of the sort's arithmetic."""
