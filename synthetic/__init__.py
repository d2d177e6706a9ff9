"""Seeded synthetic inputs (no method arithmetic); see synthetic/inputs.py."""
