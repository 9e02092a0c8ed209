namespace sellb { int set_error(int c, const char*, ...) { return c; } }
