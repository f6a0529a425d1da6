cd scripts/ubench && ./stream
