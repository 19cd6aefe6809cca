/* ktune_b200 executable: the command-line front end is compiled into
 * libktune_b200.so (csrc/tools/ktune_b200.cpp, entry ktune_cli_main). */
int ktune_cli_main(int argc, char** argv);

int main(int argc, char** argv) { return ktune_cli_main(argc, argv); }
