cd scripts/ubench && ./pipes
