"""Test-side tools that use the oracle (only tests/ may import it); not collected by pytest."""
